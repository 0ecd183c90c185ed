python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "x_new||--coarse 0" "x_px2|PSFS_LIB=variants/px2/libpsfs.so|--coarse 0"
done > gpurun_out/ab_r02zn.txt 2>&1
