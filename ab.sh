mkdir -p gpurun_out
: > gpurun_out/ab_summary.txt
run() { # name lib extra-args
  PSFS_LIB=$2 timeout 300 python bench.py --no-e2e --no-cpu-baseline $3 > gpurun_out/ab_$1.log 2>&1
  python - "$1" >> gpurun_out/ab_summary.txt <<'PY'
import json, sys
n = sys.argv[1]
try:
    j = json.loads(open(f"gpurun_out/ab_{n}.log").read().strip().splitlines()[-1])
    r = j["roofline"]; iso = r.get("isolated_serial") or {}
    print(f"{n:24s} fps={j['value']:9.0f} step={j['ms_per_step']*1e3:7.1f}us  vox={r['avg_launch_us']:6.1f} s1={r['other_kernel']['avg_launch_us']:6.1f} frac={r['frac']:.3f} iso_s1={iso.get('k_likelihood',{}).get('avg_launch_us',0):6.1f} iso_vox={iso.get('k_voxel',{}).get('avg_launch_us',0):6.1f}")
except Exception as e:
    print(n, "FAILED", e)
PY
}
L=paper_1311_6811_b200/libpsfs.so
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
run f16_ovl $L "--batch 32"
run f16_ser $L "--batch 32 --overlap -1"
run f16_ovl_b64 $L "--batch 64 --pool 64"
run f16_ser_b64 $L "--batch 64 --pool 64 --overlap -1"
cat gpurun_out/ab_summary.txt
