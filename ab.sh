mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r01.json 2>gpurun_out/bench_r01.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r01.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --profile --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_likelihood|k_voxel" -s 6 -c 2 -o gpurun_out/prof_r01 python bench.py --steps 3 --warmup 3 --profile --no-e2e > /dev/null 2>&1
nvidia-smi -q -d CLOCK > gpurun_out/clocks_r01.txt 2>&1
