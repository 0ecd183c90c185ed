python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "x_new||--coarse 0" "x_head|PSFS_LIB=variants/head/libpsfs.so|--coarse 0" "b128||--batch 128 --pool 128" "b64||"
done > gpurun_out/ab_r02w.txt 2>&1
python scripts/c5_leg.py C5 C4 > gpurun_out/c5_new.txt 2>&1
PSFS_LIB=variants/gu4/libpsfs.so python scripts/c5_leg.py C5 C4 > gpurun_out/c5_gu4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_smooth.py -x -q > gpurun_out/ab_r02w_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02w_tests.log
