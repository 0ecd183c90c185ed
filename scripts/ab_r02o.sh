python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "pf2|PSFS_LIB=variants/pf2/libpsfs.so|" "pf3|PSFS_LIB=variants/pf3/libpsfs.so|" "pf4|PSFS_LIB=variants/pf4/libpsfs.so|"
done > gpurun_out/ab_r02o.txt 2>&1
