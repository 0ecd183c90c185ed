python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "nw4|PSFS_LIB=variants/nw4/libpsfs.so|" "nw4kz8|PSFS_LIB=variants/nw4/libpsfs.so|--kz 8" "nw4kz2|PSFS_LIB=variants/nw4/libpsfs.so|--kz 2"
done > gpurun_out/ab_r02p.txt 2>&1
PSFS_LIB=variants/nw4/libpsfs.so timeout 600 python -m pytest tests/test_gpu_coarse.py -x -q > gpurun_out/ab_r02p_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02p_tests.log
