"""Shared helpers for the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np


def unpack_bits(words, nvox):
    w = np.ascontiguousarray(np.asarray(words).astype(np.uint32))
    return np.unpackbits(w.view(np.uint8), bitorder="little")[:nvox].astype(bool)


def gpu_run(scene, frames_list, params=None, fuse=8, roi=True, rank=0, world=1, logodds=True,
            device=0):
    """Run the CUDA path through the ABI on a list of uint8 frame sets
    ([ncam, H, W, 3] numpy each); returns numpy (L [n, nslab], bits [n, nwords])."""
    import torch

    from paper_1311_6811_b200 import from_scene
    rec = from_scene(scene, params, device=device, rank=rank, world=world)
    rec.set_max_fuse(fuse)
    rec.set_roi_enabled(roi)
    n = len(frames_list)
    fr = torch.from_numpy(np.stack(frames_list)).cuda(device)
    L, B = rec.alloc_outputs(n, logodds=logodds, bits=True)
    rec.reconstruct_batch(fr, n, logodds=L, bits=B)
    torch.cuda.synchronize(device)
    out = dict(bits=B.cpu().numpy().view(np.uint32), rec=rec)
    out["L"] = L.cpu().numpy() if logodds else None
    return out


def assert_parity(L_gpu, bits_gpu_words, orc, nvox_slab, word0=0, tau=0.5, tol_L=1e-4, band=1e-4):
    """BASELINE.json north_star bar: log-odds within tol_L absolute; occupancy
    bit-exact except voxels whose oracle posterior is within `band` of tau
    (counted and returned)."""
    stats = {}
    if L_gpu is not None:
        err = np.abs(L_gpu.astype(np.float64) - orc["L"])
        stats["max_abs_err_L"] = float(err.max())
        assert err.max() <= tol_L, f"log-odds error {err.max()} > {tol_L}"
    b_g = unpack_bits(np.asarray(bits_gpu_words)[word0:], nvox_slab)
    b_o = unpack_bits(orc["bits"], nvox_slab)
    mism = b_g != b_o
    amb = np.abs(orc["post"] - tau) < band
    stats["bit_mismatches"] = int(mism.sum())
    stats["ambiguous_voxels"] = int(amb.sum())
    stats["occupied"] = int(b_o.sum())
    bad = mism & ~amb
    assert not bad.any(), f"{int(bad.sum())} occupancy bits differ outside the ambiguity band"
    return stats
