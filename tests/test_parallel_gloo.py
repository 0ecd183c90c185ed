"""Host-side logic of the multi-GPU partition (paper_1311_6811_b200/parallel.py),
run as real world_size > 1 process groups on CPU with the gloo backend.

The per-rank compute here is the CPU oracle restricted to the rank's z-slab
(test infrastructure standing in for the rank's GPU); what is under test is
the partition rule, the word alignment of the slabs and the bitmask
all-gather that assembles the full grid on every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1311_6811_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("n", [32, 128, 256, 512, 1024])
def test_slabs_partition_the_grid(n):
    for world in (1, 2, 4, 8):
        bounds = [parallel.slab_bounds(n, world, r) for r in range(world)]
        assert bounds[0][0] == 0 and bounds[-1][1] == n
        for (a0, a1), (b0, b1) in zip(bounds, bounds[1:]):
            assert a1 == b0 and a0 < a1
        parallel.check_partition(n, n, n, world)
        words = [parallel.slab_words(n, n, n, world, r) for r in range(world)]
        assert words[0][0] == 0 and words[-1][1] == n * n * n // 32
        assert all(w[1] - w[0] == words[0][1] - words[0][0] for w in words)


def test_partition_rejects_unaligned():
    with pytest.raises(ValueError):
        parallel.check_partition(32, 32, 30, 4)     # zlen % world
    with pytest.raises(ValueError):
        parallel.check_partition(3, 5, 8, 8)        # slab of 15 voxels is not whole words


def test_frame_parallel_assignment():
    for nframes in (1, 7, 64, 300):
        for world in (1, 2, 4, 8):
            got = sorted(f for r in range(world) for f in parallel.frame_indices(nframes, world, r))
            assert got == list(range(nframes))


def _worker(rank, world, port, nframes, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from synth.scene import make_frames, make_scene
        s = make_scene("C1")
        g = s.grid
        k0, k1 = parallel.slab_bounds(g.zlen, world, rank)
        w0, w1 = parallel.slab_words(g.xlen, g.ylen, g.zlen, world, rank)
        bits = torch.zeros((nframes, g.nwords), dtype=torch.int32)
        for f in range(nframes):
            fr = make_frames(s, f)
            part = oracle.scene_reconstruct(s, fr, k0=k0, k1=k1)
            bits[f, w0:w1] = torch.from_numpy(part["bits"].view(np.int32))
        parallel.allgather_bits(bits, g.xlen, g.ylen, g.zlen, world, rank)
        result_q.put((rank, bits.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_zslab_allgather_assembles_full_grid(world):
    """Each rank fills only its slab's words; after the all-gather every rank
    holds exactly the single-process full-grid bitmask, for every frame."""
    import oracle
    from synth.scene import make_frames, make_scene
    nframes = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nframes, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = make_scene("C1")
    for f in range(nframes):
        full = oracle.scene_reconstruct(s, make_frames(s, f))["bits"].view(np.int32)
        for r in range(world):
            assert np.array_equal(results[r][f], full), (r, f)


def _handles_worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = bytes([rank]) * 64  # stands in for this rank's cudaIpcMemHandle_t
        result_q.put((rank, parallel.exchange_handles(h, world)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_exchange_handles_rank_order(world):
    """The fused exchange's one host collective: every rank receives every
    rank's IPC handle, in rank order (what psfs_peer_open expects)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_handles_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [bytes([r]) * 64 for r in range(world)]
    for r in range(world):
        assert results[r] == want


def _halo_worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plane, slices, nf = 6, 3, 2
        # rank r's slab: value = 1000 * frame + global slice index * 10 + x
        k0 = rank * slices
        sums = torch.tensor([[1000 * f + (k0 + k) * 10 + x for k in range(slices) for x in range(plane)]
                             for f in range(nf)], dtype=torch.int32)
        lo, hi = parallel.exchange_halos(sums, plane, world, rank)
        result_q.put((rank, (None if lo is None else lo.numpy(), None if hi is None else hi.numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_exchange_halos_neighbour_slices(world):
    """NEXT-1 on z-slabs: rank r receives slice k0 - 1 (the last slice of rank
    r - 1) and slice k1 (the first of rank r + 1), none at the volume's ends."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plane, slices, nf = 6, 3, 2
    for r in range(world):
        lo, hi = res[r]
        k0, k1 = r * slices, (r + 1) * slices
        want = lambda k: np.array([[1000 * f + k * 10 + x for x in range(plane)] for f in range(nf)])
        assert (lo is None) == (r == 0) and (hi is None) == (r == world - 1)
        if lo is not None:
            assert np.array_equal(lo, want(k0 - 1))
        if hi is not None:
            assert np.array_equal(hi, want(k1))
