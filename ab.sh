mkdir -p gpurun_out
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_color.json 2>gpurun_out/bench_color.err; tail -1 gpurun_out/bench_color.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['color'], j['surface'], j['smooth'])"; tail -3 gpurun_out/bench_color.err
