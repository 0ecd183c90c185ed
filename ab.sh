mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "sixteen_frame_pass" > gpurun_out/pytest_fs.log 2>&1; tail -3 gpurun_out/pytest_fs.log
