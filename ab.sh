mkdir -p gpurun_out
summ() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); r=d['roofline']; k={r['kernel']:r, r['other_kernel']['kernel']:r['other_kernel']}
print('$1', round(d['value']), 'fps  s1', round(k['k_likelihood']['avg_launch_us'],1), 'us  s2', round(k['k_voxel']['avg_launch_us'],1),'us')" 2>&1 | tail -1; }
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
timeout 300 $B --stage1 0 > gpurun_out/ab_s0.log 2>&1; summ gpurun_out/ab_s0.log
timeout 300 ncu --set full --clock-control none -k "regex:k_likelihood" -s 3 -c 1 -o gpurun_out/prof_rows $B --steps 3 --warmup 3 --profile > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
