# Build libpsfs.so from a git revision (default HEAD) into variants/<name>/ for A/B runs.
# usage: scripts/build_head_variant.sh NAME [REV] [-DMACRO ...]
set -e
name=$1; rev=${2:-HEAD}; shift 2 || true
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_1311_6811_b200/csrc include | tar -x -C "$tmp"
mkdir -p "$root/variants/$name"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -shared \
  -Xcompiler -fPIC,-ffp-contract=off "$@" -o "$root/variants/$name/libpsfs.so" \
  "$tmp/paper_1311_6811_b200/csrc/psfs_api.cu" "$tmp/paper_1311_6811_b200/csrc/psfs_kernels.cu" \
  "$tmp/paper_1311_6811_b200/csrc/psfs_next3.cu"
rm -rf "$tmp"
echo "$root/variants/$name/libpsfs.so"
