python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "memonly|PSFS_LIB=variants/memonly/libpsfs.so|"
done > gpurun_out/ab_r02zc.txt 2>&1
