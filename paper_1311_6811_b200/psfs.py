"""Thin ctypes binding of the C ABI in include/psfs.h (argument marshalling only).

Every step of the PSFS path runs in the sm_100a kernels of libpsfs.so; this
module converts torch tensors / numpy arrays into the pointers and sizes the
ABI takes.  There is no CPU fallback: if libpsfs.so is missing or the device
is not a CUDA GPU, every call raises.

PyTorch supplies device memory (torch.empty(..., device='cuda')), streams
(torch.cuda.current_stream().cuda_stream) and, in parallel.py, process groups.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PSFS_LIB overrides the library (A/B experiments with variant builds only)
LIB_PATH = os.environ.get("PSFS_LIB", os.path.join(_HERE, "libpsfs.so"))

PSFS_OK = 0
STATUS = {0: "PSFS_OK", 1: "PSFS_EINVAL", 2: "PSFS_EDEGENERATE", 3: "PSFS_EDIM", 4: "PSFS_ECOUNT",
          5: "PSFS_ESTATE", 6: "PSFS_ECUDA", 7: "PSFS_ENOMEM", 8: "PSFS_ELIMIT",
          9: "PSFS_ETIMEOUT"}
MAX_CAMERAS = 64
MAX_BATCH = 16
MAX_PEERS = 8
IPC_HANDLE_BYTES = 64

# Every symbol include/psfs.h declares (checked by tests/test_abi.py).
EXPORTS = ["psfs_default_params", "psfs_create", "psfs_set_cameras", "psfs_set_background",
           "psfs_reconstruct", "psfs_reconstruct_batch", "psfs_reconstruct_host", "psfs_destroy",
           "psfs_status_string", "psfs_last_error", "psfs_slab", "psfs_debug_matrices",
           "psfs_debug_terms", "psfs_debug_roi", "psfs_set_roi_enabled", "psfs_set_max_fuse",
           "psfs_last_launch_count", "psfs_set_profiling", "psfs_kernel_times",
           "psfs_fast_rcp_enabled", "psfs_debug_rcp_check", "psfs_probe_l1_bandwidth",
           "psfs_set_stage1_path", "psfs_set_voxel_tile", "psfs_set_overlap",
           "psfs_set_carve", "psfs_surface", "psfs_smooth_threshold", "psfs_peer_alloc",
           "psfs_peer_open", "psfs_reconstruct_peer", "psfs_peer_status", "psfs_color",
           "psfs_train_background", "psfs_probe_gather_bandwidth", "psfs_set_coarse",
           "psfs_coarse_plan", "psfs_coarse_status", "psfs_debug_codes", "psfs_set_host_upload",
           "psfs_set_input", "psfs_reconstruct_sums", "psfs_smooth_sums", "psfs_reconstruct_smoothed",
           "psfs_mc_create", "psfs_mc_attach", "psfs_mc_bind", "psfs_mc_release", "psfs_roi_pixels"]
MC_HANDLE_BYTES = 64
SAMPLE_NEAREST = 0
SAMPLE_BILINEAR = 1
MAX_COARSE = 64


class PsfsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Grid(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("spacing", C.c_double),
                ("xlen", C.c_int32), ("ylen", C.c_int32), ("zlen", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("occlusion_prior", C.c_double), ("voxel_prior", C.c_double),
                ("threshold", C.c_double), ("sigma_floor", C.c_double)]


class Dist(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32)]


_lib = None


def lib():
    """Load libpsfs.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, d = C.c_void_p, C.c_int32, C.c_double
        L.psfs_default_params.argtypes = [C.POINTER(Params)]
        L.psfs_default_params.restype = None
        L.psfs_create.argtypes = [C.POINTER(Grid), C.POINTER(Params), C.POINTER(Dist), C.POINTER(vp)]
        L.psfs_set_cameras.argtypes = [vp, i32, vp, vp, vp]
        L.psfs_set_background.argtypes = [vp, i32, i32, i32, vp, vp]
        L.psfs_reconstruct.argtypes = [vp, vp, vp, vp, vp]
        L.psfs_reconstruct_batch.argtypes = [vp, i32, vp, vp, vp, vp]
        L.psfs_reconstruct_host.argtypes = [vp, i32, vp, vp, vp, vp]
        L.psfs_destroy.argtypes = [vp]
        L.psfs_destroy.restype = None
        L.psfs_status_string.argtypes = [C.c_int]
        L.psfs_status_string.restype = C.c_char_p
        L.psfs_last_error.argtypes = [vp]
        L.psfs_last_error.restype = C.c_char_p
        L.psfs_slab.argtypes = [vp, C.POINTER(i32), C.POINTER(i32)]
        L.psfs_debug_matrices.argtypes = [vp, vp]
        L.psfs_debug_terms.argtypes = [vp, vp, vp, vp]
        L.psfs_debug_roi.argtypes = [vp, vp]
        L.psfs_set_roi_enabled.argtypes = [vp, i32]
        L.psfs_set_max_fuse.argtypes = [vp, i32]
        L.psfs_set_stage1_path.argtypes = [vp, i32]
        L.psfs_set_voxel_tile.argtypes = [vp, i32, i32]
        L.psfs_set_overlap.argtypes = [vp, i32, i32]
        L.psfs_set_carve.argtypes = [vp, i32]
        L.psfs_surface.argtypes = [vp, vp, vp, vp, C.c_int64, vp, vp]
        L.psfs_smooth_threshold.argtypes = [vp, vp, vp, vp, vp]
        L.psfs_last_launch_count.argtypes = [vp]
        L.psfs_set_profiling.argtypes = [vp, i32]
        L.psfs_kernel_times.argtypes = [vp, vp, vp, i32]
        L.psfs_fast_rcp_enabled.argtypes = [vp]
        L.psfs_debug_rcp_check.argtypes = [C.c_float, C.c_float, C.POINTER(C.c_int64)]
        L.psfs_probe_l1_bandwidth.argtypes = [C.POINTER(C.c_double)]
        L.psfs_probe_gather_bandwidth.argtypes = [C.c_int64, i32, i32, C.POINTER(C.c_double)]
        L.psfs_peer_alloc.argtypes = [vp, i32, C.POINTER(vp), vp]
        L.psfs_peer_open.argtypes = [vp, vp]
        L.psfs_reconstruct_peer.argtypes = [vp, i32, vp, vp, vp]
        L.psfs_peer_status.argtypes = [vp, vp]
        L.psfs_color.argtypes = [vp, vp, vp, vp, C.c_int64, d, vp, vp, vp]
        L.psfs_train_background.argtypes = [vp, i32, i32, vp, vp, vp, i32, vp]
        L.psfs_set_coarse.argtypes = [vp, i32, i32, i32, C.c_int64]
        L.psfs_coarse_plan.argtypes = [C.POINTER(Params), i32, vp, C.POINTER(d)]
        L.psfs_coarse_status.argtypes = [vp, C.POINTER(i32), C.POINTER(C.c_int64), i32]
        L.psfs_debug_codes.argtypes = [vp, vp, vp, vp]
        L.psfs_set_host_upload.argtypes = [vp, i32]
        L.psfs_set_input.argtypes = [vp, i32, i32]
        L.psfs_reconstruct_sums.argtypes = [vp, i32, vp, vp, vp, vp]
        L.psfs_smooth_sums.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp]
        L.psfs_reconstruct_smoothed.argtypes = [vp, i32, vp, vp, vp, vp]
        L.psfs_mc_create.argtypes = [vp, i32, vp]
        L.psfs_mc_attach.argtypes = [vp, vp]
        L.psfs_mc_bind.argtypes = [vp, C.POINTER(vp)]
        L.psfs_mc_release.argtypes = [vp]
        L.psfs_roi_pixels.argtypes = [vp, C.POINTER(C.c_int64)]
        _lib = L
    return _lib


def default_params() -> dict:
    p = Params()
    lib().psfs_default_params(C.byref(p))
    return dict(occlusion_prior=p.occlusion_prior, voxel_prior=p.voxel_prior,
                threshold=p.threshold, sigma_floor=p.sigma_floor)


def coarse_plan(params: dict | None = None, ncam: int = 8) -> dict:
    """Host-only psfs_coarse_plan: the code bracket for these params."""
    p = Params()
    lib().psfs_default_params(C.byref(p))
    for k, v in (params or {}).items():
        setattr(p, k, float(v))
    out = np.zeros(7, np.int32)
    eps = C.c_double()
    rc = lib().psfs_coarse_plan(C.byref(p), int(ncam), out.ctypes.data, C.byref(eps))
    if rc != PSFS_OK:
        raise PsfsError(rc, "psfs_coarse_plan")
    return dict(ok=bool(out[0]), sh=int(out[1]), bias=int(out[2]), wc=int(out[3]), K0=int(out[4]),
                K1=int(out[5]), Tq=int(out[6]), eps=eps.value)


def _ptr_array(ptrs):
    arr = (C.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
    return arr


def _dev_ptr(t, dtype=None):
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"expected dtype {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


@dataclass
class GridSpec:
    origin: tuple
    spacing: float
    xlen: int
    ylen: int
    zlen: int

    @property
    def nvox(self):
        return self.xlen * self.ylen * self.zlen

    @property
    def nwords(self):
        return (self.nvox + 31) // 32


class Reconstructor:
    """One library handle (psfs_create ... psfs_destroy) on one CUDA device."""

    def __init__(self, grid, params: dict | None = None, device: int | None = None,
                 rank: int = 0, world: int = 1):
        import torch
        self._h = None
        g = Grid((C.c_double * 3)(*[float(x) for x in grid.origin]), float(grid.spacing),
                 int(grid.xlen), int(grid.ylen), int(grid.zlen))
        p = Params()
        lib().psfs_default_params(C.byref(p))
        for k, v in (params or {}).items():
            setattr(p, k, float(v))
        if device is None:
            device = torch.cuda.current_device()
        dist = Dist(int(device), int(rank), int(world))
        h = C.c_void_p()
        rc = lib().psfs_create(C.byref(g), C.byref(p), C.byref(dist), C.byref(h))
        if rc != PSFS_OK:
            raise PsfsError(rc, "psfs_create failed")
        self._h = h
        self.grid = GridSpec(tuple(grid.origin), float(grid.spacing), int(grid.xlen),
                             int(grid.ylen), int(grid.zlen))
        self.device = int(device)
        self.rank, self.world = int(rank), int(world)
        k0, k1 = C.c_int32(), C.c_int32()
        lib().psfs_slab(h, C.byref(k0), C.byref(k1))
        self.k0, self.k1 = k0.value, k1.value
        self.ncam = 0
        self.widths = self.heights = None
        self.channels = 3
        self.sampling = SAMPLE_NEAREST

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if self._h is not None:
            lib().psfs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc != PSFS_OK:
            msg = lib().psfs_last_error(self._h).decode() if self._h else ""
            raise PsfsError(rc, f"{what}: {msg}")

    # -- setup -------------------------------------------------------------
    def set_cameras(self, P, widths, heights):
        P = np.ascontiguousarray(np.asarray(P, np.float64).reshape(-1, 12))
        W = np.ascontiguousarray(np.asarray(widths, np.int32))
        H = np.ascontiguousarray(np.asarray(heights, np.int32))
        self._check(lib().psfs_set_cameras(self._h, P.shape[0], P.ctypes.data, W.ctypes.data,
                                           H.ctypes.data), "psfs_set_cameras")
        self.ncam = P.shape[0]
        self.widths, self.heights = W.copy(), H.copy()
        self.npix = int((W.astype(np.int64) * H).sum())

    def set_input(self, channels: int = 3, sampling: int = SAMPLE_NEAREST):
        """NEXT-3: 3 (RGB) or 1 (grayscale) channels per pixel; nearest-pixel or
        bilinear SLM sampling (include/psfs.h psfs_set_input).  A channel change
        discards the background models."""
        self._check(lib().psfs_set_input(self._h, int(channels), int(sampling)), "psfs_set_input")
        self.channels, self.sampling = int(channels), int(sampling)

    def set_background(self, cam, mean, sigma):
        mean = np.ascontiguousarray(np.asarray(mean, np.float32))
        sigma = np.ascontiguousarray(np.asarray(sigma, np.float32))
        if mean.ndim != 3 or mean.shape != sigma.shape or mean.shape[2] != self.channels:
            raise ValueError(f"mean/sigma must be [H, W, {self.channels}] float32")
        self._check(lib().psfs_set_background(self._h, int(cam), mean.shape[1], mean.shape[0],
                                              mean.ctypes.data, sigma.ctypes.data),
                    "psfs_set_background")

    def train_background(self, cam, frames, install=True, outputs=True, stream=None):
        """NEXT-3: train camera `cam`'s background model on the GPU from a uint8
        CUDA tensor [n, H, W, 3] of background frames; install=True makes it the
        camera's model.  Returns (mean, sigma) float32 CUDA tensors or None."""
        import torch
        if not (isinstance(frames, torch.Tensor) and frames.is_cuda and frames.dtype == torch.uint8
                and frames.is_contiguous() and frames.dim() == 4):
            raise TypeError("frames must be a contiguous uint8 CUDA tensor [n, H, W, channels]")
        n = frames.shape[0]
        per = frames[0].numel()
        ptrs = _ptr_array([frames.data_ptr() + f * per for f in range(n)])
        mean = sigma = None
        if outputs:
            mean = torch.empty(frames.shape[1:], dtype=torch.float32, device=frames.device)
            sigma = torch.empty_like(mean)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_train_background(self._h, int(cam), int(n), ptrs,
                                                _dev_ptr(mean, torch.float32),
                                                _dev_ptr(sigma, torch.float32), int(bool(install)),
                                                s), "psfs_train_background")
        return mean, sigma

    def set_max_fuse(self, fmax: int):
        self._check(lib().psfs_set_max_fuse(self._h, int(fmax)), "psfs_set_max_fuse")

    def set_coarse(self, mode: int = 1, max_frames: int = MAX_COARSE, min_frames: int = 0,
                   fix_capacity: int = 0):
        """Coarse passes for bits-only calls: 0 off, 1 on (default), 2 every
        voxel-frame resolved exactly (test mode); frames per pass 1..64; calls
        with fewer than min_frames frames stay exact (0 = default 16); fix-up
        list entries (0 = default 2^20)."""
        self._check(lib().psfs_set_coarse(self._h, int(mode), int(max_frames), int(min_frames),
                                          int(fix_capacity)), "psfs_set_coarse")

    def coarse_status(self, reset: bool = False):
        """(applies to bits-only calls, voxel-frames resolved exactly since the last reset)."""
        a, n = C.c_int32(), C.c_int64()
        self._check(lib().psfs_coarse_status(self._h, C.byref(a), C.byref(n), int(bool(reset))),
                    "psfs_coarse_status")
        return bool(a.value), int(n.value)

    def set_host_upload(self, mode: int):
        """psfs_reconstruct_host uploads: 1 zero-copy kernel for mapped pinned frames
        (default), 0 DMA 2-D copies."""
        self._check(lib().psfs_set_host_upload(self._h, int(mode)), "psfs_set_host_upload")

    def set_carve(self, on: bool):
        """Bits-only early exit (exact bitmask; ignored when log-odds are requested)."""
        self._check(lib().psfs_set_carve(self._h, int(bool(on))), "psfs_set_carve")

    def set_overlap(self, on: bool, voxel_blocks_per_sm: int = 0):
        self._check(lib().psfs_set_overlap(self._h, int(bool(on)), int(voxel_blocks_per_sm)),
                    "psfs_set_overlap")

    def set_voxel_tile(self, ty: int, kz: int):
        self._check(lib().psfs_set_voxel_tile(self._h, int(ty), int(kz)), "psfs_set_voxel_tile")

    def set_stage1_path(self, path: int):
        """0 one pixel/thread (default), 1 TMA ring, 2 pipelined, 3 four pixels/thread,
        4 warp-row loads (see include/psfs.h)."""
        self._check(lib().psfs_set_stage1_path(self._h, int(path)), "psfs_set_stage1_path")

    def set_roi_enabled(self, on):
        """True: rectangles + per-row spans (default); False: whole images;
        2: rectangles only (A/B)."""
        self._check(lib().psfs_set_roi_enabled(self._h, 2 if on == 2 else int(bool(on))), "psfs_set_roi_enabled")

    # -- outputs -------------------------------------------------------------
    @property
    def nslab(self):
        return self.grid.xlen * self.grid.ylen * (self.k1 - self.k0)

    def alloc_outputs(self, nframes=1, logodds=True, bits=True):
        import torch
        dev = torch.device("cuda", self.device)
        L = torch.empty((nframes, self.nslab), dtype=torch.float32, device=dev) if logodds else None
        B = torch.zeros((nframes, self.grid.nwords), dtype=torch.int32, device=dev) if bits else None
        return L, B

    # -- the hot path ---------------------------------------------------------
    def _frame_ptrs(self, frames, nframes):
        """frames: a uint8 CUDA tensor [nframes, ncam, H, W, 3] (or [ncam, H, W, 3]
        when nframes == 1), a nested list [f][c] of [H, W, 3] tensors, or a
        pointer table from frame_pointers() (reused as is)."""
        import torch
        if isinstance(frames, C.Array):
            if len(frames) < nframes * self.ncam:
                raise ValueError("pointer table too short")
            return frames
        ptrs = []
        if isinstance(frames, torch.Tensor):
            t = frames
            if t.dim() == 4:
                t = t.unsqueeze(0)
            if t.dtype != torch.uint8 or not t.is_cuda or not t.is_contiguous():
                raise TypeError("frames must be a contiguous uint8 CUDA tensor")
            if t.shape[0] != nframes or t.shape[1] != self.ncam:
                raise ValueError("frames shape mismatch")
            base = t.data_ptr()
            per_cam = t[0, 0].numel()
            for f in range(nframes):
                for c in range(self.ncam):
                    ptrs.append(base + (f * self.ncam + c) * per_cam)
        else:
            for f in range(nframes):
                row = frames[f] if nframes > 1 or isinstance(frames[0], (list, tuple)) else frames
                for c in range(self.ncam):
                    ptrs.append(_dev_ptr(row[c], torch.uint8))
        return _ptr_array(ptrs)

    def frame_pointers(self, frames, nframes: int):
        """The HOST table of nframes * ncam device frame pointers the ABI takes,
        built once (e.g. outside a timed loop) and passed back as `frames`; the
        tensors it points into must stay alive."""
        return self._frame_ptrs(frames, nframes)

    def reconstruct_batch(self, frames, nframes: int, logodds=None, bits=None, stream=None):
        """Enqueue both stages for nframes frame sets on `stream` (default: the
        current torch stream).  Outputs are caller-owned CUDA tensors:
        logodds float32 [nframes, nslab], bits int32 [nframes, nwords]."""
        import torch
        fp = self._frame_ptrs(frames, nframes)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        Lp = _dev_ptr(logodds, torch.float32)
        Bp = _dev_ptr(bits, torch.int32)
        if logodds is not None and logodds.numel() < nframes * self.nslab:
            raise ValueError("logodds too small")
        if bits is not None and bits.numel() < nframes * self.grid.nwords:
            raise ValueError("bits too small")
        self._check(lib().psfs_reconstruct_batch(self._h, int(nframes), fp, Lp, Bp, s),
                    "psfs_reconstruct_batch")

    # -- fused z-slab exchange (include/psfs.h psfs_peer_*) --------------------
    def peer_alloc(self, nframes: int):
        """Allocate this rank's exchange buffer (nframes full-grid bitmasks);
        returns (bits int32 CUDA tensor [nframes, nwords] viewing it, the
        IPC handle bytes to hand to every other rank)."""
        import torch
        ptr = C.c_void_p()
        hbuf = C.create_string_buffer(IPC_HANDLE_BYTES)
        self._check(lib().psfs_peer_alloc(self._h, int(nframes), C.byref(ptr), hbuf),
                    "psfs_peer_alloc")
        nwords = self.grid.nwords

        class _View:  # __cuda_array_interface__ over the library-owned buffer
            __cuda_array_interface__ = {"shape": (int(nframes), nwords), "typestr": "<i4",
                                        "data": (int(ptr.value), False), "version": 2,
                                        "strides": None}
        with torch.cuda.device(self.device):
            bits = torch.as_tensor(_View(), device=torch.device("cuda", self.device))
        self._peer_bits = bits
        return bits, hbuf.raw

    # -- NVLS multicast bitmask buffer (include/psfs.h psfs_mc_*) ----------------
    def mc_create(self, nframes: int) -> bytes:
        """Size the multicast buffer; rank 0 creates the object and returns its
        handle bytes (other ranks: zeros)."""
        hbuf = C.create_string_buffer(MC_HANDLE_BYTES)
        self._check(lib().psfs_mc_create(self._h, int(nframes), hbuf), "psfs_mc_create")
        self._mc_frames = int(nframes)
        return hbuf.raw

    def mc_attach(self, handle: bytes):
        buf = C.create_string_buffer(bytes(handle), MC_HANDLE_BYTES)
        self._check(lib().psfs_mc_attach(self._h, buf), "psfs_mc_attach")

    def mc_bind(self):
        """Bind this device's replica; returns an int32 CUDA tensor [nframes,
        nwords] viewing it (the full-grid bitmasks after psfs_reconstruct_peer)."""
        import torch
        ptr = C.c_void_p()
        self._check(lib().psfs_mc_bind(self._h, C.byref(ptr)), "psfs_mc_bind")
        nwords = self.grid.nwords

        class _View:
            __cuda_array_interface__ = {"shape": (self._mc_frames, nwords), "typestr": "<i4",
                                        "data": (int(ptr.value), False), "version": 2, "strides": None}
        with torch.cuda.device(self.device):
            bits = torch.as_tensor(_View(), device=torch.device("cuda", self.device))
        self._mc_bits = bits
        return bits

    def mc_release(self):
        self._mc_bits = None
        self._check(lib().psfs_mc_release(self._h), "psfs_mc_release")

    def peer_open(self, handles):
        """handles: list of world IPC handle byte strings in rank order."""
        if len(handles) != self.world or any(len(x) != IPC_HANDLE_BYTES for x in handles):
            raise ValueError("need world handles of IPC_HANDLE_BYTES each")
        buf = C.create_string_buffer(b"".join(handles), IPC_HANDLE_BYTES * self.world)
        self._check(lib().psfs_peer_open(self._h, buf), "psfs_peer_open")

    def reconstruct_peer(self, frames, nframes: int, logodds=None, stream=None):
        """Both stages with the bitmask bytes stored into every rank's exchange
        buffer, between device-side entry and exit barriers (all ranks call it)."""
        import torch
        fp = self._frame_ptrs(frames, nframes)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        if logodds is not None and logodds.numel() < nframes * self.nslab:
            raise ValueError("logodds too small")
        self._check(lib().psfs_reconstruct_peer(self._h, int(nframes), fp,
                                                _dev_ptr(logodds, torch.float32), s),
                    "psfs_reconstruct_peer")

    def peer_status(self, stream=None):
        """Synchronize and raise PsfsError(PSFS_ETIMEOUT) if a barrier timed out."""
        import torch
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_peer_status(self._h, s), "psfs_peer_status")

    def reconstruct(self, frames, logodds=None, bits=None, stream=None):
        import torch
        fp = self._frame_ptrs(frames, 1)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_reconstruct(self._h, fp, _dev_ptr(logodds, torch.float32),
                                           _dev_ptr(bits, torch.int32), s), "psfs_reconstruct")

    def reconstruct_host(self, frames_host, nframes: int, logodds_host=None, bits_host=None,
                         stream=None):
        """End-to-end call with HOST buffers (pinned for overlap): the library
        copies frames in, runs both stages and copies results out, overlapping
        the transfers of one frame group with the compute of the previous one.
        frames_host: uint8 tensor/ndarray [nframes, ncam, H, W, 3] in host memory;
        outputs: host float32 [nframes, nslab] / int32 [nframes, nwords]."""
        import torch
        def hp(x):
            if x is None:
                return None
            if isinstance(x, torch.Tensor):
                assert not x.is_cuda and x.is_contiguous()
                return x.data_ptr()
            assert x.flags["C_CONTIGUOUS"]
            return x.ctypes.data
        base = hp(frames_host)
        per_cam = int(self.widths[0]) * int(self.heights[0]) * self.channels
        if not (self.widths == self.widths[0]).all() or not (self.heights == self.heights[0]).all():
            raise ValueError("reconstruct_host helper assumes equal camera sizes")
        ptrs = _ptr_array([base + i * per_cam for i in range(nframes * self.ncam)])
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_reconstruct_host(self._h, int(nframes), ptrs, hp(logodds_host),
                                                hp(bits_host), s), "psfs_reconstruct_host")

    def surface(self, bits, surface_bits=None, indices=None, count=None, stream=None):
        """Surface voxels (NEXT-2) of this handle's slab from a full-grid bitmask
        (int32 CUDA tensor of nwords).  Returns (count tensor [1] int64, indices
        tensor or None, surface_bits or None); everything stays on the device."""
        import torch
        dev = torch.device("cuda", self.device)
        if count is None:
            count = torch.zeros(1, dtype=torch.int64, device=dev)
        cap = 0 if indices is None else indices.numel()
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_surface(self._h, _dev_ptr(bits, torch.int32),
                                       _dev_ptr(surface_bits, torch.int32),
                                       _dev_ptr(indices, torch.int64), cap,
                                       _dev_ptr(count, torch.int64), s), "psfs_surface")
        return count, indices, surface_bits

    def smooth_threshold(self, logodds, smoothed=None, bits=None, stream=None):
        """NEXT-1: box-filtered posterior and its threshold bits from a full-grid
        log-odds tensor (float32 CUDA, nvox).  Outputs are caller-owned tensors."""
        import torch
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_smooth_threshold(self._h, _dev_ptr(logodds, torch.float32),
                                                _dev_ptr(smoothed, torch.float32),
                                                _dev_ptr(bits, torch.int32), s),
                    "psfs_smooth_threshold")
        return smoothed, bits

    def reconstruct_sums(self, frames, nframes: int, sums, bits=None, stream=None):
        """NEXT-1 step 1: both stages with the exact int32 sums S (int32 CUDA tensor
        [nframes, nslab]) as the per-voxel output; optional unsmoothed bits."""
        import torch
        fp = self._frame_ptrs(frames, nframes)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        if sums.numel() < nframes * self.nslab:
            raise ValueError("sums too small")
        self._check(lib().psfs_reconstruct_sums(self._h, int(nframes), fp, _dev_ptr(sums, torch.int32),
                                                _dev_ptr(bits, torch.int32), s), "psfs_reconstruct_sums")

    def smooth_sums(self, nframes: int, sums, halo_lo=None, halo_hi=None, smoothed=None, bits=None,
                    stream=None):
        """NEXT-1 step 2: posterior 3x3x3 box average > tau from the sums; z-slab
        handles pass the neighbours' boundary slices (int32 [nframes, xlen*ylen])."""
        import torch
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_smooth_sums(self._h, int(nframes), _dev_ptr(sums, torch.int32),
                                           _dev_ptr(halo_lo, torch.int32), _dev_ptr(halo_hi, torch.int32),
                                           _dev_ptr(smoothed, torch.float32), _dev_ptr(bits, torch.int32), s),
                    "psfs_smooth_sums")
        return smoothed, bits

    def reconstruct_smoothed(self, frames, nframes: int, smoothed=None, bits=None, stream=None):
        """NEXT-1 merged with reconstruction (world-1 handles): smoothed posterior
        (float32 [nframes, nvox], nullable) and its threshold bits."""
        import torch
        fp = self._frame_ptrs(frames, nframes)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_reconstruct_smoothed(self._h, int(nframes), fp, _dev_ptr(smoothed, torch.float32),
                                                    _dev_ptr(bits, torch.int32), s), "psfs_reconstruct_smoothed")
        return smoothed, bits

    # -- introspection ----------------------------------------------------------
    def debug_terms(self, frames, stream=None):
        import torch
        out = torch.empty(self.npix, dtype=torch.int32, device=torch.device("cuda", self.device))
        fp = self._frame_ptrs(frames, 1)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_debug_terms(self._h, fp, out.data_ptr(), s), "psfs_debug_terms")
        return out

    def debug_codes(self, frames, stream=None):
        """Coarse stage 1 of one frame set over whole images: uint8 codes (c + bias)."""
        import torch
        out = torch.empty(self.npix, dtype=torch.uint8, device=torch.device("cuda", self.device))
        fp = self._frame_ptrs(frames, 1)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_debug_codes(self._h, fp, out.data_ptr(), s), "psfs_debug_codes")
        return out

    def matrices(self):
        out = np.empty((self.ncam, 12), np.float32)
        self._check(lib().psfs_debug_matrices(self._h, out.ctypes.data), "psfs_debug_matrices")
        return out

    def roi_pixels(self) -> int:
        """Stage-1 pixels of one frame set (per-row spans, or rectangles)."""
        v = C.c_int64()
        self._check(lib().psfs_roi_pixels(self._h, C.byref(v)), "psfs_roi_pixels")
        return int(v.value)

    def roi(self):
        out = np.empty((self.ncam, 4), np.int32)
        self._check(lib().psfs_debug_roi(self._h, out.ctypes.data), "psfs_debug_roi")
        return out

    def color(self, frames, indices, count=None, rgb=None, nviews=None, slm_gate=0.5, stream=None):
        """NEXT-4 voxel colour of one frame set ([ncam, H, W, 3] uint8 CUDA
        tensor) at int64 CUDA `indices`; count: optional int64 CUDA tensor [1]
        (e.g. from surface()), else all of `indices`.  Returns (rgb float32
        [capacity, 3], nviews int32 [capacity]) CUDA tensors."""
        import torch
        dev = torch.device("cuda", self.device)
        cap = int(indices.numel())
        if count is None:
            count = torch.tensor([cap], dtype=torch.int64, device=dev)
        if rgb is None:
            rgb = torch.empty((cap, 3), dtype=torch.float32, device=dev)
        if nviews is None:
            nviews = torch.empty(cap, dtype=torch.int32, device=dev)
        fp = self._frame_ptrs(frames, 1)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        self._check(lib().psfs_color(self._h, fp, _dev_ptr(indices, torch.int64),
                                     _dev_ptr(count, torch.int64), cap, float(slm_gate),
                                     _dev_ptr(rgb, torch.float32), _dev_ptr(nviews, torch.int32),
                                     s), "psfs_color")
        return rgb, nviews

    def set_profiling(self, on: bool):
        self._check(lib().psfs_set_profiling(self._h, int(bool(on))), "psfs_set_profiling")

    def kernel_times(self, reset=True):
        """{'k_likelihood': (ms, launches), 'k_voxel': (ms, launches)} since last reset."""
        ms = np.zeros(2, np.float64)
        n = np.zeros(2, np.int64)
        self._check(lib().psfs_kernel_times(self._h, ms.ctypes.data, n.ctypes.data, int(reset)),
                    "psfs_kernel_times")
        return {"k_likelihood": (float(ms[0]), int(n[0])), "k_voxel": (float(ms[1]), int(n[1]))}

    @property
    def fast_rcp(self) -> bool:
        return bool(lib().psfs_fast_rcp_enabled(self._h))

    @property
    def last_launch_count(self):
        return int(lib().psfs_last_launch_count(self._h))


def probe_gather_bandwidth(table_bytes: int = 64 << 20, sectors_per_line: int = 2,
                           blocks_per_sm: int = 3) -> float:
    """Bytes/s of a voxel kernel's gather pattern on the current device
    (psfs_probe_gather_bandwidth): sectors_per_line 2 = k_voxel16 (lane pairs on
    two-sector records, 3 blocks/SM), 1 = k_voxel_c8 (one sector per lane, 2 blocks/SM)."""
    v = C.c_double()
    rc = lib().psfs_probe_gather_bandwidth(int(table_bytes), int(sectors_per_line), int(blocks_per_sm),
                                           C.byref(v))
    if rc != PSFS_OK:
        raise PsfsError(rc, "psfs_probe_gather_bandwidth")
    return float(v.value)


def debug_rcp_check(lo: float, hi: float) -> int:
    """Mismatches between the fast reciprocal and RN(1/w) over every float in [lo, hi)."""
    n = C.c_int64()
    rc = lib().psfs_debug_rcp_check(float(lo), float(hi), C.byref(n))
    if rc != PSFS_OK:
        raise PsfsError(rc, "psfs_debug_rcp_check")
    return int(n.value)


def probe_l1_bandwidth() -> float:
    """Measured L1 load bandwidth (bytes/s) of the current device."""
    v = C.c_double()
    rc = lib().psfs_probe_l1_bandwidth(C.byref(v))
    if rc != PSFS_OK:
        raise PsfsError(rc, "psfs_probe_l1_bandwidth")
    return float(v.value)


def from_scene(scene, params=None, device=None, rank=0, world=1, sampling=SAMPLE_NEAREST) -> Reconstructor:
    """Build a Reconstructor for a synth.Scene-like object (grid, P, widths,
    heights, mu, sigma; the channel count is mu's last axis)."""
    r = Reconstructor(scene.grid, params, device, rank, world)
    nch = int(np.asarray(scene.mu).shape[-1])
    if nch != 3 or sampling != SAMPLE_NEAREST:
        r.set_input(nch, sampling)
    r.set_cameras(scene.P, scene.widths, scene.heights)
    for c in range(scene.ncam):
        r.set_background(c, scene.mu[c], scene.sigma[c])
    return r
