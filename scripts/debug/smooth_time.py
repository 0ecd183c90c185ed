import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
from synth.scene import make_scene, make_frames
from paper_1311_6811_b200 import from_scene
s = make_scene("C2")
fr = torch.from_numpy(np.stack([make_frames(s, f % 8) for f in range(16)])).cuda()
rec = from_scene(s)
_, B = rec.alloc_outputs(16, logodds=False)
for _ in range(3):
    rec.reconstruct_smoothed(fr, 16, bits=B)
torch.cuda.synchronize()
