python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "nosum|PSFS_LIB=variants/nosum/libpsfs.so|" "hints3|PSFS_LIB=variants/hints3/libpsfs.so|"
done > gpurun_out/ab_r02y.txt 2>&1
