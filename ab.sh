mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); r=d['roofline']; o=r['other_kernel']
print(round(d['value']), 'fps', r['kernel'], round(r['frac'],3), round(r['avg_launch_us'],1), '|', o['kernel'], round(o['frac'],3), round(o['avg_launch_us'],1), 'e2e', round(d['e2e']['value']), 'carve', round(d['carve']['value']))"
