python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "a3m5|PSFS_LIB=variants/a3m5/libpsfs.so|" "a3m4|PSFS_LIB=variants/a3m4/libpsfs.so|" "a2m5|PSFS_LIB=variants/a2m5/libpsfs.so|"
done > gpurun_out/ab_r02s.txt 2>&1
PSFS_LIB=variants/a3m5/libpsfs.so timeout 900 python -m pytest tests/test_gpu_coarse.py -x -q > gpurun_out/ab_r02s_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02s_tests.log
