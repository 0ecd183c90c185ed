mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "host" > gpurun_out/pytest_host.log 2>&1; tail -3 gpurun_out/pytest_host.log
python bench.py --no-cpu-baseline --no-zslab > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err
tail -1 gpurun_out/bench_e2e.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['e2e'])"
