# A/B: stage-1 hints once per thread, stage-2 3/4 blocks per SM; then ncu --set full of the new default
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "new||" "hints2|PSFS_LIB=variants/hints2/libpsfs.so|" "minb3|PSFS_LIB=variants/minb3/libpsfs.so|" "minb4|PSFS_LIB=variants/minb4/libpsfs.so|"
done > gpurun_out/ab_r02n.txt 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k "regex:k_likelihood_c8p|k_voxel_c8w|k_fixup_c8" -s 6 -c 3 -f -o gpurun_out/r02n_headline python bench.py --steps 3 --warmup 3 --profile --no-e2e --no-cpu-baseline --no-zslab --no-secondaries > gpurun_out/r02n_ncu.log 2>&1
echo NCU_EXIT=$? >> gpurun_out/r02n_ncu.log
