"""NEXT-1 merged (psfs_reconstruct_smoothed) on C2, 64 frames per call, with per-kernel
device times (psfs_set_profiling): A/B of k_box_sums variants.  usage: python scripts/smooth_leg.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1311_6811_b200 import from_scene  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
stream = torch.cuda.current_stream(dev)
flush = (torch.empty(256 << 20, dtype=torch.uint8, device=dev), torch.empty(256 << 20, dtype=torch.uint8, device=dev))
scene, frames = bench.make_workload("C2", 64)
fr = torch.from_numpy(frames).to(dev)
rs = from_scene(scene, device=0)
_, Bs = rs.alloc_outputs(64, logodds=False)
tab = rs.frame_pointers(fr[:64], 64)
rs.reconstruct_smoothed(tab, 64, bits=Bs, stream=stream)
torch.cuda.synchronize(dev)
ms = bench.timed_calls(lambda k: rs.reconstruct_smoothed(tab, 64, bits=Bs, stream=stream), 10, stream, flush)
print(json.dumps({"frames_per_s": 64 * len(ms) / (sum(ms) / 1e3), "call_ms": bench.step_stats(ms)}))
