mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_smooth.py -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
