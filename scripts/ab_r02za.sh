python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "x_new||--coarse 0" "x_xg0|PSFS_LIB=variants/xg0/libpsfs.so|--coarse 0" "x_head|PSFS_LIB=variants/head/libpsfs.so|--coarse 0" "s1_new||--batch 1 --pool 16 --steps 50" "s1_head|PSFS_LIB=variants/head/libpsfs.so|--batch 1 --pool 16 --steps 50"
done > gpurun_out/ab_r02za.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_coarse.py -x -q > gpurun_out/ab_r02za_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02za_tests.log
