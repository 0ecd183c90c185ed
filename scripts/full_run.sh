# Full GPU round check: build, pytest -m gpu, smoke(), bench (default), ncu launch list and --set full of the headline.
# usage: bash scripts/full_run.sh TAG
T=${1:-r02x}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputest.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/${T}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > gpurun_out/${T}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo BENCH_EXIT=$? >> gpurun_out/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --profile --no-e2e --no-cpu-baseline --no-zslab --no-secondaries > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k "regex:k_likelihood_c8p|k_voxel_c8w|k_fixup_c8" -s 6 -c 3 -f -o gpurun_out/${T}_headline python bench.py --steps 3 --warmup 3 --profile --no-e2e --no-cpu-baseline --no-zslab --no-secondaries > gpurun_out/${T}_ncu_full.log 2>&1
echo DONE
