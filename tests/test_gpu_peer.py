"""The fused z-slab bitmask exchange (psfs_peer_alloc / psfs_peer_open /
psfs_reconstruct_peer) with real CUDA IPC mappings:
`world` processes share GPU 0 (one process per rank, exactly as one process
per GPU, only the peer stores stay on one device), torch.distributed (gloo)
moves the IPC handles once, stage 2 stores every slab byte into every rank's
buffer and device-side barriers order the exchange.  Every rank must end up
with the single-handle full-grid bitmask, bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth.scene import Grid, make_frames, make_scene
from tests.helpers import gpu_run

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _scene(kind):
    if kind == "C1":
        return make_scene("C1")
    # xlen % 8 != 0: ragged rows, the kernel ORs bits into peer words atomically
    g = Grid((-1000.0, -1000.0, 0.0), 2000.0 / 36, 36, 40, 16)
    return make_scene("C1", grid=g, W=66, H=50)


def _worker(rank, world, port, kind, nframes, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1311_6811_b200 import PsfsError
        from paper_1311_6811_b200.parallel import ZSlabReconstructor
        torch.cuda.set_device(0)
        s = _scene(kind)
        z = ZSlabReconstructor(s, rank=rank, world=world, device=0, peer=True, max_frames=nframes)
        fr = torch.from_numpy(np.stack([make_frames(s, f) for f in range(nframes)])).cuda()
        if mode == "timeout":
            # rank 1 never enters the exchange: rank 0's barriers must give up
            # (bounded spin) and report PSFS_ETIMEOUT instead of hanging
            code = None
            if rank == 0:
                z.reconstruct_batch(fr, nframes)
                try:
                    z.rec.peer_status()
                except PsfsError as e:
                    code = e.code
            dist.barrier()
            q.put((rank, code))
            return
        out = []
        for rep in range(2):  # twice: the entry barrier protects the reused buffers
            frames = fr if rep == 0 else fr.flip(0).contiguous()
            bits = z.reconstruct_batch(frames, nframes)
            z.rec.peer_status()
            out.append(bits.cpu().numpy().copy())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(world, kind, nframes, mode="ok"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, nframes, mode, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,kind,nframes", [(2, "C1", 3), (4, "C1", 17), (2, "ragged", 2)])
def test_fused_exchange_gives_every_rank_the_full_grid(world, kind, nframes):
    res = _run(world, kind, nframes)
    s = _scene(kind)
    frames = [make_frames(s, f) for f in range(nframes)]
    ref = gpu_run(s, frames, fuse=16)["bits"]
    ref_flip = ref[::-1]
    for r in range(world):
        assert np.array_equal(res[r][0].view(np.uint32), ref), r
        assert np.array_equal(res[r][1].view(np.uint32), ref_flip), r


def test_barrier_times_out_instead_of_hanging():
    from paper_1311_6811_b200.psfs import STATUS
    res = _run(2, "C1", 1, mode="timeout")
    assert STATUS[res[0]] == "PSFS_ETIMEOUT"


def _bench_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import argparse
        import bench
        torch.cuda.set_device(0)
        s = make_scene("C1")
        fr = torch.from_numpy(np.stack([make_frames(s, f) for f in range(16)])).cuda()
        args = argparse.Namespace(steps=2, warmup=1)
        out = bench.zslab_bench(args, s, fr, rank, world, 0, torch.device("cuda", 0),
                                torch.cuda.current_stream(), variants=(("fused_peer", True),))
        assert out["world"] == world and out["frames_per_call"] == 16
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_bench_zslab_section():
    """bench.py's N > 1 z-slab measurement (fused variant) runs and reports."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r]["fused_peer"]["frames_per_s"] > 0
