# A/B of the round-2 session-3 variants (headline bench only), then the coarse GPU suites
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "base|PSFS_LIB=variants/base/libpsfs.so|" "nofast|PSFS_LIB=variants/c8w_nofast/libpsfs.so|" "nobulk|PSFS_LIB=variants/c8p_nobulk/libpsfs.so|" "hoist|PSFS_LIB=variants/c8w_hoist/libpsfs.so|"
done > gpurun_out/ab_r02m.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_parity.py tests/test_gpu_pads.py tests/test_gpu_peer.py -x -q > gpurun_out/ab_r02m_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02m_tests.log
