"""Multi-GPU partition of the PSFS path.

One process per GPU (torchrun), torch.distributed for the plumbing:

* frame-parallel ("weak" scaling, configs C2/C3/C5 sequences): rank r takes
  frames r, r+N, ...; each rank is an independent single-GPU handle, no
  collective on the data path (voxels and frames are independent, PAPER.md:228
  "the procedures for each voxel has nothing to do with others", and the
  uniform foreground model makes frames independent, R#17).
* z-slab (config C4): rank r owns slices [r*zlen/N, (r+1)*zlen/N) of the grid
  (the library's psfs_dist), runs stage 1 only on the pixel rectangle its slab
  projects into, stage 2 on its slab, and the full occupancy bitmask is
  assembled on every rank either
  - fused (peer=True, the default on GPUs of one node): stage 2 stores each
    ballot byte of the slab into every rank's exchange buffer through CUDA IPC
    peer mappings (NVLink / NVSwitch), ordered by device-side barriers --
    no separate collective; torch.distributed only moves the IPC handles once;
  - or by one in-place all-gather of the per-slab words (NCCL over NVLink on
    GPUs; gloo in the CPU tests).
  Log-odds stay sharded.
* NEXT-1 on z-slabs (reconstruct_smoothed): the 3x3x3 box filter of the
  posterior needs one slice of each neighbouring slab; every rank computes
  its slab's exact int32 sums (psfs_reconstruct_sums), sends its first slice
  to rank - 1 and its last to rank + 1 and receives their boundary slices
  (exchange_halos: point-to-point send/recv, NCCL on GPUs, gloo on CPU
  tensors), then smooths and thresholds its slab (psfs_smooth_sums); the
  smoothed bitmask is all-gathered like the plain one.

The slab rule here is the same pure function the library applies
(k0 = zlen*rank//world); tests check both agree.
"""
from __future__ import annotations

import os


def slab_bounds(zlen: int, world: int, rank: int):
    """[k0, k1) of rank's z-slab (integer rule of psfs_create)."""
    return zlen * rank // world, zlen * (rank + 1) // world


def check_partition(xlen: int, ylen: int, zlen: int, world: int):
    """z-slab mode needs equal slabs of whole bitmask words."""
    if zlen % world:
        raise ValueError(f"zlen={zlen} not divisible by world={world}")
    if (xlen * ylen * (zlen // world)) % 32:
        raise ValueError("slab is not a whole number of 32-bit words")


def slab_words(xlen, ylen, zlen, world, rank):
    k0, k1 = slab_bounds(zlen, world, rank)
    return xlen * ylen * k0 // 32, xlen * ylen * k1 // 32


def frame_indices(nframes: int, world: int, rank: int):
    """Frame-parallel assignment: rank r takes r, r+N, r+2N, ..."""
    return list(range(rank, nframes, world))


def allgather_bits(bits, xlen, ylen, zlen, world, rank, group=None):
    """In-place all-gather of slab words: bits is an int32 tensor [nframes, nwords]
    (or [nwords]) holding this rank's slab words; afterwards every rank holds the
    full grid.  One collective per frame row (all_gather_into_tensor)."""
    import torch
    import torch.distributed as dist
    check_partition(xlen, ylen, zlen, world)
    if world == 1:
        return bits
    b = bits if bits.dim() == 2 else bits.unsqueeze(0)
    nwords = xlen * ylen * zlen // 32
    chunk = nwords // world
    for f in range(b.shape[0]):
        row = b[f, :nwords]
        mine = row[rank * chunk:(rank + 1) * chunk]
        if row.is_cuda:
            dist.all_gather_into_tensor(row, mine, group=group)
        else:  # gloo has no in-place all_gather_into_tensor: gather a list
            parts = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine.clone(), group=group)
            row.copy_(torch.cat(parts))
    return bits


def exchange_halos(sums, plane: int, world: int, rank: int, group=None):
    """One-slice halo exchange between neighbouring z-slabs (NEXT-1 on slabs):
    sums is this rank's [nframes, nslab] int32 tensor; rank r sends slice k0
    (its first plane) to r - 1 and slice k1 - 1 (its last) to r + 1, and
    receives slice k0 - 1 from r - 1 (halo_lo) and slice k1 from r + 1
    (halo_hi).  Returns (halo_lo, halo_hi), None at the volume's boundary.
    One batch of isend/irecv (NCCL for CUDA tensors, gloo for CPU)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return None, None
    b = sums if sums.dim() == 2 else sums.unsqueeze(0)
    first = b[:, :plane].contiguous()
    last = b[:, b.shape[1] - plane:].contiguous()
    lo = torch.empty_like(first) if rank > 0 else None
    hi = torch.empty_like(last) if rank < world - 1 else None
    # one batch (ncclGroupStart/End under NCCL): separate sends posted before the
    # matching receives would serialise on the pair's stream and deadlock
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, first, rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, lo, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, last, rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, hi, rank + 1, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return lo, hi


def env_rank_world():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def exchange_handles(handle: bytes, world: int, group=None):
    """All-gather one IPC handle per rank (host objects; any backend)."""
    import torch.distributed as dist
    if world == 1:
        return [handle]
    out = [None] * world
    dist.all_gather_object(out, handle, group=group)
    return out


class ZSlabReconstructor:
    """A z-slab handle plus the bitmask exchange: fused peer stores (peer=True)
    or an NCCL all-gather of the slab words (peer=False)."""

    def __init__(self, scene, params=None, rank=None, world=None, device=None, group=None,
                 peer=False, max_frames=16, multicast=False):
        from .psfs import from_scene
        r, w, local = env_rank_world()
        self.rank = r if rank is None else rank
        self.world = w if world is None else world
        g = scene.grid
        check_partition(g.xlen, g.ylen, g.zlen, self.world)
        self.grid = g
        self.group = group
        self.rec = from_scene(scene, params, device=local if device is None else device,
                              rank=self.rank, world=self.world)
        self.peer = peer
        self.bits = None
        self.multicast = False
        if peer:
            # host collectives at setup only: every rank maps every other rank's
            # buffer; a failure on any rank makes every rank raise (no rank is
            # left waiting in a collective or a device barrier)
            try:
                self.bits, h = self.rec.peer_alloc(max_frames)
            except Exception:
                h = b""
            handles = exchange_handles(h, self.world, group)
            if any(not x for x in handles):
                raise RuntimeError("psfs_peer_alloc failed on rank(s) "
                                   f"{[r for r, x in enumerate(handles) if not x]}")
            try:
                self.rec.peer_open(handles)
                ok = b"1"
            except Exception:
                ok = b""
            oks = exchange_handles(ok, self.world, group)
            if not all(oks):
                raise RuntimeError("psfs_peer_open failed on rank(s) "
                                   f"{[r for r, x in enumerate(oks) if not x]}")
            self.multicast = bool(multicast) and self._setup_multicast(max_frames)

    def _setup_multicast(self, max_frames):
        """NVLS multicast buffer for the bitmask (include/psfs.h psfs_mc_*): rank 0
        creates, every rank attaches its device, then binds its replica, with a
        host agreement after each step; any failure on any rank releases it
        everywhere and the exchange keeps the per-rank peer stores."""
        def agree(ok):
            return all(exchange_handles(b"1" if ok else b"", self.world, self.group))

        try:
            h = self.rec.mc_create(max_frames)
            ok = True
        except Exception:
            h, ok = b"", False
        handles = exchange_handles(h, self.world, self.group)
        if agree(ok):
            try:
                self.rec.mc_attach(handles[0])
                ok = True
            except Exception:
                ok = False
            if agree(ok):  # every device added before any replica is bound
                try:
                    bits = self.rec.mc_bind()
                    ok = True
                except Exception:
                    ok = False
                if agree(ok):
                    self.bits = bits
                    return True
        try:
            self.rec.mc_release()
        except Exception:
            pass
        return False

    def reconstruct_smoothed(self, frames, nframes, smoothed=None, bits=None, stream=None, gather=True):
        """NEXT-1 on the z-slab partition: sums of this slab, halo exchange with
        the neighbours, smoothing + threshold of the slab, and (gather) the
        smoothed bitmask all-gathered so every rank holds the full grid.
        smoothed: float32 [nframes, nslab] (nullable); bits: int32 [nframes,
        nwords].  Returns bits."""
        import torch
        import torch.distributed as dist
        g = self.grid
        plane = g.xlen * g.ylen
        dev = torch.device("cuda", self.rec.device)
        sums = torch.empty((nframes, self.rec.nslab), dtype=torch.int32, device=dev)
        self.rec.reconstruct_sums(frames, nframes, sums, stream=stream)
        lo = hi = None
        if self.world > 1:
            # NCCL: stream-ordered after the sums (torch's current stream); gloo
            # moves CPU tensors only (the .cpu() copy synchronizes)
            cpu = dist.get_backend(self.group) != "nccl"
            lo, hi = exchange_halos(sums.cpu() if cpu else sums, plane, self.world, self.rank, self.group)
            if cpu:
                lo = lo.to(dev) if lo is not None else None
                hi = hi.to(dev) if hi is not None else None
        self.rec.smooth_sums(nframes, sums, lo, hi, smoothed=smoothed, bits=bits, stream=stream)
        if gather and bits is not None and self.world > 1:
            cpu = dist.get_backend(self.group) != "nccl"
            if cpu:
                b = bits.cpu()
                allgather_bits(b, g.xlen, g.ylen, g.zlen, self.world, self.rank, self.group)
                bits.copy_(b.to(dev))
            else:
                allgather_bits(bits, g.xlen, g.ylen, g.zlen, self.world, self.rank, self.group)
        return bits

    def reconstruct_batch(self, frames, nframes, logodds=None, bits=None, stream=None,
                          gather=True):
        """peer mode: the full-grid bitmasks land in self.bits[:nframes] on every
        rank (stream-ordered, no host synchronisation); `bits` is ignored."""
        if self.peer:
            self.rec.reconstruct_peer(frames, nframes, logodds=logodds, stream=stream)
            return self.bits[:nframes]
        self.rec.reconstruct_batch(frames, nframes, logodds=logodds, bits=bits, stream=stream)
        if gather and bits is not None:
            g = self.grid
            allgather_bits(bits, g.xlen, g.ylen, g.zlen, self.world, self.rank, self.group)
        return bits
