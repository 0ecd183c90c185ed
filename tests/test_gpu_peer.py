"""The fused z-slab bitmask exchange (psfs_peer_alloc / psfs_peer_open /
psfs_reconstruct_peer) with real CUDA IPC mappings:
`world` processes share GPU 0 (one process per rank, exactly as one process
per GPU, only the peer stores stay on one device), torch.distributed (gloo)
moves the IPC handles once, stage 2 stores every slab byte into every rank's
buffer and device-side barriers order the exchange.  Every rank's assembled
full-grid bitmask is checked against the CPU oracle frame by frame (bits exact
outside the 1e-4 posterior band; BASELINE.json north_star), and against the
single-handle run bit for bit.  The all-gather variant (peer=False) runs the
same slab handles with the words gathered by parallel.allgather_bits (gloo on
CPU tensors here: NCCL refuses two ranks on one device)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from synth.scene import Grid, make_frames, make_scene
from tests.helpers import assert_parity, gpu_run, unpack_bits

NTHREADS = max(1, len(os.sched_getaffinity(0)))

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
        z = ZSlabReconstructor(s, rank=rank, world=world, device=0, peer=(mode not in ("allgather", "smooth")),
                               max_frames=nframes)
        fr = torch.from_numpy(np.stack([make_frames(s, f) for f in range(nframes)])).cuda()
        if mode == "smooth":  # NEXT-1 on slabs: sums, halo exchange (gloo), smoothing, all-gather
            bits = torch.zeros((nframes, s.grid.nwords), dtype=torch.int32, device="cuda")
            sm = torch.empty((nframes, z.rec.nslab), dtype=torch.float32, device="cuda")
            z.reconstruct_smoothed(fr, nframes, smoothed=sm, bits=bits)
            torch.cuda.synchronize()
            q.put((rank, (bits.cpu().numpy().copy(), sm.cpu().numpy().copy(), z.rec.k0, z.rec.k1)))
            return
        if mode == "allgather":
            from paper_1311_6811_b200.parallel import allgather_bits
            out = []
            for lo in (False, True):  # bits only (coarse passes when >= 16 frames) / with log-odds (exact)
                L, B = z.rec.alloc_outputs(nframes, logodds=lo)
                z.reconstruct_batch(fr, nframes, logodds=L, bits=B, gather=False)
                torch.cuda.synchronize()
                Bc = B.cpu()
                g = s.grid
                allgather_bits(Bc, g.xlen, g.ylen, g.zlen, world, rank)
                out.append(Bc.numpy().copy())
            q.put((rank, out))
            return
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


def _oracle_bits_check(s, frames, words_per_frame):
    """Every frame's full-grid bitmask against the oracle (A5 parity)."""
    for f, fr in enumerate(frames):
        orc = oracle.scene_reconstruct(s, fr, nthreads=NTHREADS)
        assert_parity(None, words_per_frame[f], orc, s.grid.nvox)


@pytest.mark.parametrize("world,kind,nframes", [(2, "C1", 3), (4, "C1", 17), (2, "ragged", 2)])
def test_fused_exchange_gives_every_rank_the_full_grid(world, kind, nframes):
    """3 frames: exact path; 17 frames on C1: one coarse pass with the fix-up
    patching every rank's buffer; ragged rows: atomic ORs into peer words."""
    res = _run(world, kind, nframes)
    s = _scene(kind)
    frames = [make_frames(s, f) for f in range(nframes)]
    ref = gpu_run(s, frames, fuse=16)["bits"]
    ref_flip = ref[::-1]
    for r in range(world):
        got = res[r][0].view(np.uint32)
        _oracle_bits_check(s, frames, got)
        _oracle_bits_check(s, frames[::-1], res[r][1].view(np.uint32))
        assert np.array_equal(got, ref), r
        assert np.array_equal(res[r][1].view(np.uint32), ref_flip), r


@pytest.mark.parametrize("world,nframes", [(2, 3), (4, 17)])
def test_allgather_exchange_against_oracle(world, nframes):
    """The all-gather variant of the z-slab exchange: every rank's gathered
    bitmask (bits-only call and log-odds call) against the oracle."""
    res = _run(world, "C1", nframes, mode="allgather")
    s = _scene("C1")
    frames = [make_frames(s, f) for f in range(nframes)]
    for r in range(world):
        for out in res[r]:
            _oracle_bits_check(s, frames, out.view(np.uint32))


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


@pytest.mark.parametrize("world,nframes", [(2, 2), (4, 3)])
def test_zslab_smoothing_against_oracle(world, nframes):
    """NEXT-1 across ranks: each rank's smoothed slab and the all-gathered
    smoothed bitmask against the oracle's box filter of the full posterior."""
    res = _run(world, "C1", nframes, mode="smooth")
    s = _scene("C1")
    g = s.grid
    plane = g.xlen * g.ylen
    for f in range(nframes):
        orc = oracle.scene_reconstruct(s, make_frames(s, f), nthreads=NTHREADS)
        sm_o, bits_o = oracle.smooth_threshold(orc["post"], g, 0.5)
        for r in range(world):
            bits, sm, k0, k1 = res[r]
            assert np.abs(sm[f].astype(np.float64) - sm_o[plane * k0: plane * k1]).max() <= 1e-5
            mism = unpack_bits(bits[f].view(np.uint32), g.nvox) != unpack_bits(bits_o, g.nvox)
            assert not (mism & ~(np.abs(sm_o - 0.5) < 1e-4)).any()


@pytest.mark.parametrize("kind,nframes", [("C1", 3), ("C1", 17), ("ragged", 2)])
def test_multicast_exchange_single_rank(kind, nframes):
    """The NVLS multicast variant of the fused exchange (psfs_mc_*), exercised
    on the one GPU a call gets: a multicast object with one device, bitmask
    words as multimem stores, ragged rows as multimem OR reductions into
    cleared words, coarse fix-ups as multimem OR / AND.  The bitmask in the
    replica equals the plain path's and meets the oracle.  Where the driver /
    fabric has no multicast, the fallback (peer stores) is what is checked."""
    from paper_1311_6811_b200.parallel import ZSlabReconstructor
    s = _scene(kind)
    frames = [make_frames(s, f) for f in range(nframes)]
    z = ZSlabReconstructor(s, rank=0, world=1, device=0, peer=True, max_frames=nframes, multicast=True)
    # where the driver / fabric refuses the multicast object (cuMulticastCreate on
    # the single-GPU test boxes), setup must fall back cleanly to the peer stores,
    # and the same checks run on that path
    print("multicast" if z.multicast else "multicast unavailable: peer-store fallback")
    fr = torch.from_numpy(np.stack(frames)).cuda()
    for rep in range(2):
        bits = z.reconstruct_batch(fr if rep == 0 else fr.flip(0).contiguous(), nframes)
        z.rec.peer_status()
        got = bits.cpu().numpy().view(np.uint32).copy()
        want = frames if rep == 0 else frames[::-1]
        ref = gpu_run(s, want, fuse=16)["bits"]
        assert np.array_equal(got, ref)
        _oracle_bits_check(s, want, got)
