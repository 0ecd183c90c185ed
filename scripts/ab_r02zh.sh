python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "head|PSFS_LIB=variants/head/libpsfs.so|" "tz8|PSFS_LIB=variants/tz8/libpsfs.so|" "tz16|PSFS_LIB=variants/tz16/libpsfs.so|" "tz32|PSFS_LIB=variants/tz32/libpsfs.so|"
done > gpurun_out/ab_r02zh.txt 2>&1
PSFS_LIB=variants/tz16/libpsfs.so timeout 900 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_peer.py -x -q > gpurun_out/ab_r02zh_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02zh_tests.log
