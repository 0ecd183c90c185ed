# ncu --set full of the exact path's kernels (k_likelihood_x4p<16>, k_voxel16) in the bench's exact step
T=${1:-r02x}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k "regex:k_likelihood_x4p|k_voxel16" -s 8 -c 2 -f -o gpurun_out/${T}_exact python bench.py --coarse 0 --steps 3 --warmup 3 --profile --no-e2e --no-cpu-baseline --no-zslab --no-secondaries > gpurun_out/${T}_exact_ncu.log 2>&1
echo NCU_EXIT=$?
