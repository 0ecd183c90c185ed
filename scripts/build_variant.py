"""Build an experiment variant of libpsfs.so into variants/<name>/ (A/B runs only).

usage: python scripts/build_variant.py NAME [-DMACRO[=V] ...]; then run with PSFS_LIB=variants/NAME/libpsfs.so
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_6811_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.ROOT, "variants", name)
os.makedirs(out, exist_ok=True)
cmd = [os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"), *b.NVCC_FLAGS, *defs, "-o",
       os.path.join(out, "libpsfs.so"), *b.SOURCES]
r = subprocess.run(cmd, capture_output=True, text=True)
open(os.path.join(out, "build.log"), "w").write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
if r.returncode:
    sys.exit(r.stderr[-3000:])
print(os.path.join(out, "libpsfs.so"))
