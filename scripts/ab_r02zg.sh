python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
for v in new box16 bz16 bz32 bz128; do
  if [ $v = new ]; then L=""; else L="PSFS_LIB=variants/$v/libpsfs.so"; fi
  echo $v $(env $L python scripts/smooth_leg.py 2>/dev/null | tail -1)
done
done > gpurun_out/ab_r02zg.txt 2>&1
for v in box16 bz32; do
PSFS_LIB=variants/$v/libpsfs.so timeout 900 python -m pytest tests/test_gpu_smooth.py -x -q > gpurun_out/ab_r02zg_tests_$v.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_r02zg_tests_$v.log
done
