# round-1 default configuration: bench line, launch list, ncu --set full of both kernels
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -1 gpurun_out/bench_default.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --profile --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_likelihood|k_voxel" -s 6 -c 2 -o gpurun_out/prof_r01 python bench.py --steps 3 --warmup 3 --profile --no-e2e --no-cpu-baseline --overlap -1 > /dev/null 2>&1
ls -la gpurun_out/prof_r01.ncu-rep gpurun_out/launches_r01.csv
