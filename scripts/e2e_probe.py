"""End-to-end probe (C2): psfs_reconstruct_host frames/s for a 64-frame step,
and the raw pinned H2D bandwidth of one large copy for comparison."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1311_6811_b200 import from_scene  # noqa: E402
from synth.scene import make_frames, make_scene  # noqa: E402

s = make_scene("C2")
B = 64
frames = np.stack([make_frames(s, f % 16) for f in range(B)])
rec = from_scene(s)
hf = torch.from_numpy(frames).pin_memory()
hb = torch.zeros((B, s.grid.nwords), dtype=torch.int32).pin_memory()
st = torch.cuda.current_stream()
for _ in range(3):
    rec.reconstruct_host(hf, B, None, hb, stream=st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(10):
    rec.reconstruct_host(hf, B, None, hb, stream=st)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"e2e {B / ms * 1e3:.0f} frames/s, {ms:.3f} ms/step")
d = torch.empty(hf.numel(), dtype=torch.uint8, device="cuda")
for _ in range(2):
    d.copy_(hf.view(-1), non_blocking=True)
torch.cuda.synchronize()
e0.record(st)
d.copy_(hf.view(-1), non_blocking=True)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"raw pinned H2D {hf.numel() / ms / 1e6:.1f} GB/s ({hf.numel() / 1e6:.0f} MB)")
