mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -k "sixteen or batch_of_16 or 29_frames or ragged or general_priors or overlapped or carve or peer or 64_frames or tile or zslab or full_size" > gpurun_out/pytest_st.log 2>&1; tail -3 gpurun_out/pytest_st.log
: > gpurun_out/ab_summary.txt
run() { # name lib extra-args
  PSFS_LIB=$2 timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-zslab $3 > gpurun_out/ab_$1.log 2>&1
  python - "$1" >> gpurun_out/ab_summary.txt <<'PY'
import json, sys
n = sys.argv[1]
try:
    j = json.loads(open(f"gpurun_out/ab_{n}.log").read().strip().splitlines()[-1])
    r = j["roofline"]; iso = r.get("isolated_serial") or {}
    print(f"{n:24s} fps={j['value']:9.0f} med={j['step_ms']['median']*1e3:.1f}  vox={r['avg_launch_us']:6.1f} s1={r['other_kernel']['avg_launch_us']:6.1f} iso_s1={iso.get('k_likelihood',{}).get('avg_launch_us',0):6.1f} iso_vox={iso.get('k_voxel',{}).get('avg_launch_us',0):6.1f} frac={r['frac']:.3f}")
except Exception as e:
    print(n, "FAILED", e)
PY
}
run stage paper_1311_6811_b200/libpsfs.so ""
run stage2 paper_1311_6811_b200/libpsfs.so ""
cat gpurun_out/ab_summary.txt
