python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "x_new||--coarse 0" "x_head|PSFS_LIB=variants/head/libpsfs.so|--coarse 0" "new||"
done > gpurun_out/ab_r02ze.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next3.py tests/test_gpu_train.py -x -q > gpurun_out/ab_r02ze_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02ze_tests.log
