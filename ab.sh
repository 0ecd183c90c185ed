mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --profile --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_likelihood|k_voxel" -s 6 -c 2 -o gpurun_out/prof_r01 python bench.py --steps 3 --warmup 3 --profile --no-e2e --overlap -1 > /dev/null 2>&1
