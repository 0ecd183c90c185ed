# full GPU suite, default bench line, launch list, ncu --set full of both kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -1 gpurun_out/bench_default.json | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print(j['value'], j['step_ms']['median'], r['avg_launch_us'], r['frac'], r['isolated_serial'], j['e2e']['value'], j['cpu_baseline']['value'], j['zslab'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --profile --no-e2e --no-cpu-baseline --no-zslab > /dev/null 2>&1
rm -f gpurun_out/prof_r01.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_likelihood|k_voxel" -s 8 -c 2 -o gpurun_out/prof_r01 python bench.py --steps 3 --warmup 3 --profile --no-e2e --no-cpu-baseline --no-zslab --overlap -1 > /dev/null 2>&1
ls -la gpurun_out/prof_r01.ncu-rep gpurun_out/launches_r01.csv
