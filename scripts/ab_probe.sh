#!/bin/bash
# A/B of libpsfs variants with scripts/coarse_probe.py, alternating, 3 rounds.
# usage: scripts/ab_probe.sh NF variantA variantB ...  ("" = the in-tree build)
nf=$1; shift
for r in 1 2 3; do
  for v in "$@"; do
    if [ "$v" = "main" ]; then unset PSFS_LIB; else export PSFS_LIB=variants/$v/libpsfs.so; fi
    echo "== $v round $r: $(python scripts/coarse_probe.py $nf 10 2>&1 | grep 'mode 1')"
  done
done
