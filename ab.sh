mkdir -p gpurun_out
summ() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); r=d['roofline']; k={r['kernel']:r, r['other_kernel']['kernel']:r['other_kernel']}
print('$1', round(d['value']), 'fps  s1', round(k['k_likelihood']['avg_launch_us'],1), 'us  s2', round(k['k_voxel']['avg_launch_us'],1),'us', 'step', round(d['ms_per_step'],3))" 2>&1 | tail -1; }
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline"
for o in -1 2 1 3; do timeout 300 $B --overlap $o > gpurun_out/ab_o$o.log 2>&1; summ gpurun_out/ab_o$o.log; done
timeout 300 $B --overlap -1 --batch 8 --pool 16 > gpurun_out/ab_b8.log 2>&1; summ gpurun_out/ab_b8.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
