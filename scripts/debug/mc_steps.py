import os, sys
sys.path.insert(0, os.getcwd())
import torch
from synth.scene import make_scene
from paper_1311_6811_b200 import from_scene
s = make_scene("C1")
rec = from_scene(s, rank=0, world=1)
for step in ("create", "attach", "bind"):
    try:
        if step == "create":
            h = rec.mc_create(4); print("create ok", h[:8].hex())
        elif step == "attach":
            rec.mc_attach(h); print("attach ok")
        else:
            b = rec.mc_bind(); print("bind ok", b.shape)
    except Exception as e:
        print(step, "FAILED:", e)
        break
