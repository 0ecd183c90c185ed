python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "spf1|PSFS_LIB=variants/spf1/libpsfs.so|"
done > gpurun_out/ab_r02zl.txt 2>&1
