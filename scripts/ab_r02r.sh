python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "head|PSFS_LIB=variants/fix1/../head/libpsfs.so|" "fix1|PSFS_LIB=variants/fix1/libpsfs.so|" "fix2|PSFS_LIB=variants/fix2/libpsfs.so|"
done > gpurun_out/ab_r02r.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_peer.py tests/test_gpu_pads.py -x -q > gpurun_out/ab_r02r_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02r_tests.log
