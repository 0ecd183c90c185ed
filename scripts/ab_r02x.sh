python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
python scripts/c5_leg.py C5 > gpurun_out/c5x_new.txt 2>&1
PSFS_LIB=variants/gu8/libpsfs.so python scripts/c5_leg.py C5 > gpurun_out/c5x_gu8.txt 2>&1
PSFS_LIB=variants/gu1/libpsfs.so python scripts/c5_leg.py C5 > gpurun_out/c5x_gu1.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab_r02x_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02x_tests.log
