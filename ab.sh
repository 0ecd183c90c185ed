mkdir -p gpurun_out
t0=$(date +%s); timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$? wall=$(( $(date +%s)-t0 ))s"; tail -2 gpurun_out/smoke.log
