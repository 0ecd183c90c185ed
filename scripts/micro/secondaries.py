"""Run the secondary calls (NEXT-1..4) a few times on C2 for an ncu launch list:
  ncu --metrics gpu__time_duration.sum --csv python scripts/micro/secondaries.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1311_6811_b200 import from_scene  # noqa: E402
from synth.scene import make_frames, make_scene  # noqa: E402

s = make_scene("C2")
rec = from_scene(s)
fr = torch.from_numpy(make_frames(s, 0)).cuda()
L, B = rec.alloc_outputs(1)
rec.reconstruct(fr, logodds=L, bits=B)
nvox = s.grid.nvox
idx = torch.empty(nvox, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
sm = torch.empty_like(L[0])
sb = torch.empty_like(B[0])
tf = torch.from_numpy(np.stack([make_frames(s, f, mode="background")[0] for f in range(32)])).cuda()
for _ in range(3):
    rec.smooth_threshold(L[0], smoothed=sm, bits=sb)
    rec.surface(B[0], indices=idx, count=cnt)
    rec.color(fr, idx, count=cnt)
    rec.train_background(0, tf, install=False)
torch.cuda.synchronize()
print("done")
