"""Debug: where does the bilinear C2 log-odds error come from?"""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
import oracle
from synth.scene import make_scene, make_frames
from paper_1311_6811_b200 import from_scene

s = make_scene("C2")
fr = make_frames(s, 0)
rec = from_scene(s, sampling=1)
L, B = rec.alloc_outputs(1)
rec.reconstruct_batch(torch.from_numpy(fr).cuda(), 1, logodds=L, bits=B)
Lg = L.cpu().numpy()[0].astype(np.float64)
slm_gpu = rec.debug_terms(torch.from_numpy(fr).cuda()).cpu().numpy().view(np.float32).astype(np.float64)
orc = oracle.scene_reconstruct(s, fr, nthreads=16, sampling="bilinear", want_slm=True)
err = np.abs(Lg - orc["L"])
print("max err", err.max(), "n>1e-5", (err > 1e-5).sum(), "n>5e-5", (err > 5e-5).sum())
# emulate with GPU SLM images in double
g = s.grid
off = 0
imgs = []
for c in range(s.ncam):
    n = s.widths[c] * s.heights[c]
    imgs.append(slm_gpu[off:off + n].reshape(s.heights[c], s.widths[c]))
    off += n
A = oracle.precompose(s.P, g.origin, g.spacing)
worst = np.argsort(err)[-5:]
for v in worst:
    i, j, k = v % g.xlen, (v // g.xlen) % g.ylen, v // (g.xlen * g.ylen)
    print("voxel", v, (i, j, k), "gpu", Lg[v], "orc", orc["L"][v], "err", err[v])
    tot_o = tot_e = 0.0
    for c in range(s.ncam):
        iv, u, vv = oracle.project_pinned_uv(A[c], s.widths[c], s.heights[c], i, j, k)
        if not iv:
            print("  cam", c, "out"); continue
        so = oracle.bilinear(orc["slm"][c], u - 0.5, vv - 0.5)
        se = oracle.bilinear(imgs[c], u - 0.5, vv - 0.5)
        x0, y0 = int(np.floor(u - 0.5)), int(np.floor(vv - 0.5))
        nb_o = orc["slm"][c][max(y0,0):y0+2, max(x0,0):x0+2]
        nb_g = imgs[c][max(y0,0):y0+2, max(x0,0):x0+2]
        to, te = np.log(2 * so), np.log(2 * se)
        tot_o += to; tot_e += te
        print(f"  cam {c} u {u:.4f} v {vv:.4f} s_orc {so:.9g} s_gpuimg {se:.9g} t_orc {to:.7f} t_gpuimg {te:.7f}")
        print("     nb_orc", nb_o.ravel(), "nb_gpu", nb_g.ravel())
    print("  sum t orc", tot_o, "emul", tot_e)
