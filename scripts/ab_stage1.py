"""A/B of the exact path's stage-1 kernels (psfs_set_stage1_path) on C2:
per-launch device time of k_likelihood and k_voxel (psfs_set_profiling events)
for 64 frames in 16-frame passes with log-odds + bits (the full-output path),
L2 flushed between calls; outputs must be bit-identical across paths."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth.scene import make_scene, make_frames
from paper_1311_6811_b200 import from_scene

paths = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,6").split(",")]
name = sys.argv[2] if len(sys.argv) > 2 else "C2"
s = make_scene(name)
nf = 64
fr = torch.from_numpy(np.stack([make_frames(s, f % 16) for f in range(nf)])).cuda()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
ref = None
res = {}
for path in paths:
    rec = from_scene(s)
    rec.set_stage1_path(path)
    rec.set_overlap(False)
    L, B = rec.alloc_outputs(nf)
    for _ in range(3):
        rec.reconstruct_batch(fr, nf, logodds=L, bits=B)
    torch.cuda.synchronize()
    rec.set_profiling(True)
    rec.kernel_times(reset=True)
    for k in range(10):
        flush.fill_(k)
        rec.reconstruct_batch(fr, nf, logodds=L, bits=B)
    torch.cuda.synchronize()
    kt = rec.kernel_times(reset=True)
    out = (L.cpu().numpy().copy(), B.cpu().numpy().copy())
    if ref is None:
        ref = out
    same = bool(np.array_equal(ref[0], out[0]) and np.array_equal(ref[1], out[1]))
    res[path] = {k: (v[0] / max(v[1], 1) * 1e3) for k, v in kt.items()}
    res[path]["identical"] = same
    print(path, json.dumps(res[path]), flush=True)
