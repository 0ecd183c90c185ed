mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_smooth.py tests/test_gpu_train.py -x -q -m gpu > gpurun_out/pytest_s.log 2>&1; tail -5 gpurun_out/pytest_s.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sec.csv python scripts/micro/secondaries.py > gpurun_out/sec.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_sec.csv
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_s.json 2>gpurun_out/bench_s.err; tail -1 gpurun_out/bench_s.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], 'smooth', j['smooth']['us_per_frame'], 'train', j['train']['us_per_camera'], 'surf', j['surface']['us_per_frame'], 'color', j['color']['us_per_frame'])"
