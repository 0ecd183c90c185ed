python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "head|PSFS_LIB=variants/head/libpsfs.so|"
done > gpurun_out/ab_r02zf.txt 2>&1
python scripts/c5_leg.py C5 > gpurun_out/c5z_new.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_peer.py tests/test_gpu_pads.py -x -q > gpurun_out/ab_r02zf_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02zf_tests.log
