mkdir -p gpurun_out
python bench.py --no-e2e --no-cpu-baseline --no-zslab > gpurun_out/bench_steps.json 2>gpurun_out/bench_steps.err
tail -1 gpurun_out/bench_steps.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['step_ms']['all'], j['clocks'])"
