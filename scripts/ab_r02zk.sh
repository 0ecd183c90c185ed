python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for rep in 1 2; do
bash scripts/ab_head.sh "kz4||" "kz8||--kz 8" "kz2||--kz 2"
done > gpurun_out/ab_r02zk.txt 2>&1
