python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2 3; do
bash scripts/ab_head.sh "new||" "fb2|PSFS_LIB=variants/fb2/libpsfs.so|"
done > gpurun_out/ab_r02zm.txt 2>&1
python scripts/c5_leg.py C5 > gpurun_out/c5zm_new.txt 2>&1
PSFS_LIB=variants/fb2/libpsfs.so python scripts/c5_leg.py C5 > gpurun_out/c5zm_fb2.txt 2>&1
