"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family of the hot path on small inputs, including the coarse
passes (PDL chain k_likelihood_c8p -> k_voxel_c8w -> k_fixup_c8 with its
self-resetting list), record-size changes (k_fill_pads), the overlapped
two-buffer schedule, the host-buffer path (k_h2d_rows), NEXT-1..4, and the
fused peer exchange with its system-scope barrier (2 processes on one GPU).

  compute-sanitizer --tool memcheck --target-processes all python scripts/sanitize_run.py

Prints one line per stage; exits non-zero on any Python-side failure."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _peer_worker(rank, world, port, nframes):
    import torch
    import torch.distributed as dist
    from paper_1311_6811_b200.parallel import ZSlabReconstructor
    from synth.scene import make_frames, make_scene
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        s = make_scene("C1")
        z = ZSlabReconstructor(s, rank=rank, world=world, device=0, peer=True, max_frames=nframes)
        fr = torch.from_numpy(np.stack([make_frames(s, f % 4) for f in range(nframes)])).cuda()
        z.reconstruct_batch(fr, nframes)
        z.rec.peer_status()
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


def main():
    import torch
    from paper_1311_6811_b200 import from_scene
    from synth.scene import Grid, make_frames, make_scene

    quick = "--quick" in sys.argv  # racecheck: smaller inputs
    dev = torch.device("cuda", 0)

    def run(scene, n, logodds, coarse_min=None, overlap=True, rec=None):
        rec = rec or from_scene(scene)
        if coarse_min is not None:
            rec.set_coarse(1, 64, coarse_min)
        rec.set_overlap(overlap, 0)
        fr = torch.from_numpy(np.stack([make_frames(scene, f % 4) for f in range(n)])).to(dev)
        L, B = rec.alloc_outputs(n, logodds=logodds)
        rec.reconstruct_batch(fr, n, logodds=L, bits=B)
        torch.cuda.synchronize()
        return rec, L, B

    c1 = make_scene("C1")
    run(c1, 3, True)
    print("exact C1 3 frames ok", flush=True)
    rec, _, _ = run(c1, 29, True)
    print("exact C1 29 frames (16+8+4+1, overlapped) ok", flush=True)
    run(c1, 17, False, coarse_min=1)
    print("coarse C1 17 frames ok", flush=True)
    run(c1, 40, False, coarse_min=1, rec=rec)
    print("coarse C1 40 frames after exact calls ok", flush=True)
    g = Grid((-6000.0, -6000.0, -3000.0), 12000.0 / 32, 32, 32, 32)
    wide = make_scene("C1", grid=g)
    rec, _, _ = run(wide, 16, True)
    run(wide, 1, True, rec=rec)
    run(wide, 20, False, rec=rec)
    run(wide, 65, False, rec=rec)
    print("record-size changes (k_fill_pads) ok", flush=True)
    g = Grid((-1000.0, -1000.0, 0.0), 2000.0 / 37, 37, 29, 23)
    ragged = make_scene("C1", grid=g, W=66, H=50)
    run(ragged, 5, True)
    print("ragged grid ok", flush=True)

    c2 = make_scene("C2")
    n2 = 16 if quick else 64
    rec, _, B = run(c2, n2, False)
    print(f"coarse C2 {n2} frames ok", flush=True)
    if not quick:
        rec2, L2, B2 = run(c2, 16, True)
        print("exact C2 16 frames ok", flush=True)
        # NEXT-1, NEXT-2, NEXT-4 on the device outputs
        sm = torch.empty_like(L2[0])
        sbits = torch.zeros(c2.grid.nwords, dtype=torch.int32, device=dev)
        rec2.smooth_threshold(L2[0], smoothed=sm, bits=sbits)
        idx = torch.empty(1 << 20, dtype=torch.int64, device=dev)
        cnt, idx, _ = rec2.surface(B2[0], indices=idx)
        fr = torch.from_numpy(make_frames(c2, 0)).to(dev)
        rec2.color(fr, idx, cnt)
        torch.cuda.synchronize()
        print("smooth / surface / color ok", flush=True)
        # NEXT-3 training
        frs = torch.from_numpy(np.stack([make_frames(c2, f, mode="background")[0] for f in range(8)])).to(dev)
        rec2.train_background(0, frs.contiguous())
        torch.cuda.synchronize()
        print("train ok", flush=True)
        # host path (zero-copy upload kernel)
        hf = torch.from_numpy(np.stack([make_frames(c2, f % 4) for f in range(20)])).pin_memory()
        Bh = torch.zeros((20, c2.grid.nwords), dtype=torch.int32).pin_memory()
        rec.reconstruct_host(hf, 20, None, Bh)
        torch.cuda.synchronize()
        print("host path ok", flush=True)

    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, 17)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=1200)
        if p.exitcode != 0:
            raise SystemExit(f"peer worker exit code {p.exitcode}")
    print("fused peer exchange (2 processes, coarse pass) ok", flush=True)


if __name__ == "__main__":
    main()
