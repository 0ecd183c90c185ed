python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "mpf1|PSFS_LIB=variants/mpf1/libpsfs.so|" "x_new||--coarse 0" "x_mpf1|PSFS_LIB=variants/xmpf1/libpsfs.so|--coarse 0"
done > gpurun_out/ab_r02v.txt 2>&1
PSFS_LIB=variants/mpf1/libpsfs.so timeout 600 python -m pytest tests/test_gpu_coarse.py -x -q > gpurun_out/ab_r02v_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02v_tests.log
PSFS_LIB=variants/xmpf1/libpsfs.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q >> gpurun_out/ab_r02v_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02v_tests.log
