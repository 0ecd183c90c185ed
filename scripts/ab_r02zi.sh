python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "mf0|PSFS_LIB=variants/mf0/libpsfs.so|" "cnv|PSFS_LIB=variants/cnv/libpsfs.so|"
done > gpurun_out/ab_r02zi.txt 2>&1
python scripts/c5_leg.py C5 C4 > gpurun_out/c5zi_new.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_coarse.py -x -q > gpurun_out/ab_r02zi_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02zi_tests.log
