mkdir -p gpurun_out
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_z.json 2>gpurun_out/bench_z.err
tail -1 gpurun_out/bench_z.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['zslab'])"; tail -2 gpurun_out/bench_z.err
