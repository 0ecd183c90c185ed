mkdir -p gpurun_out
summ() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); r=d['roofline']; k={r['kernel']:r, r['other_kernel']['kernel']:r['other_kernel']}
print('$1', round(d['value']), 'fps  s1', round(k['k_likelihood']['avg_launch_us'],1), 'us  s2', round(k['k_voxel']['avg_launch_us'],1),'us')" 2>&1 | tail -1; }
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --ty 1 --kz 4"
for p in 0 1 2; do timeout 300 $B --stage1 $p > gpurun_out/ab_s$p.log 2>&1; summ gpurun_out/ab_s$p.log; done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -m gpu -q --timeout 900 -x -k "stage1 or c2_bench or ragged or general" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
