mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_color.py -x -q -m gpu > gpurun_out/pytest_train.log 2>&1; tail -15 gpurun_out/pytest_train.log
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_train.json 2>gpurun_out/bench_train.err; tail -1 gpurun_out/bench_train.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['train'], j['color']['us_per_frame'])"; tail -3 gpurun_out/bench_train.err
