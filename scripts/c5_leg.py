"""C5 (1024^3 x 32 cameras) and C4 (512^3 x 16) coarse-pass timing through bench.variant_leg (A/B of
stage-2 variants on large camera counts).  usage: python scripts/c5_leg.py [C5|C4 ...]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
stream = torch.cuda.current_stream(dev)
flush = (torch.empty(256 << 20, dtype=torch.uint8, device=dev), torch.empty(256 << 20, dtype=torch.uint8, device=dev))

args = argparse.Namespace(steps=5)
for cfg in (sys.argv[1:] or ["C5"]):
    out, _ = bench.variant_leg(args, cfg, dev, stream, flush, 1, nframes=64, pool=1)
    print(json.dumps({cfg: {k: out[k] for k in ("frames_per_s", "ms_per_frame", "call_ms", "launches_per_call")}}))
