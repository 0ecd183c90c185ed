"""CPU oracle of the PSFS hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_1311_6811_b200``) never imports it and shares no code with it.

The arithmetic lives in ``psfs_oracle.c`` (plain loops, double precision,
pinned FP32 projection; every function cites PAPER.md).  This module only
compiles it with gcc (``-O2 -ffp-contract=off``, OpenMP for the all-core
timing mode, no fast-math) and marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "psfs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so in-tree (gcc, -O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "psfs_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Grid(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("spacing", C.c_double),
                ("xlen", C.c_int), ("ylen", C.c_int), ("zlen", C.c_int)]


class _Rig(C.Structure):
    _fields_ = [("ncam", C.c_int), ("A", C.c_void_p), ("W", C.c_void_p), ("H", C.c_void_p),
                ("p_occ", C.c_double)]


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        d, vp, i, i64 = C.c_double, C.c_void_p, C.c_int, C.c_int64
        _lib.oracle_pixel.argtypes = [vp, vp, vp, d, d, vp, vp, vp]
        _lib.oracle_view_likelihood.argtypes = [d, d, vp, vp]
        _lib.oracle_slm_image.argtypes = [i, i, vp, vp, vp, d, d, vp, vp, vp, i]
        _lib.oracle_precompose.argtypes = [vp, vp, d, vp]
        _lib.oracle_project_pinned.argtypes = [vp, i, i, i, i, i, vp, vp]
        _lib.oracle_project_pinned.restype = i
        _lib.oracle_project_exact.argtypes = [vp, vp, d, i, i, i, i, i, vp, vp]
        _lib.oracle_project_exact.restype = i
        _lib.oracle_project_pinned_batch.argtypes = [vp, i, i, i64, vp, vp]
        _lib.oracle_fuse.argtypes = [C.POINTER(_Rig), C.POINTER(_Grid), vp, vp, d, d, i, i,
                                     vp, vp, vp, i]
        _lib.oracle_fuse_sample.argtypes = [C.POINTER(_Rig), C.POINTER(_Grid), vp, vp, vp, d, d,
                                            i64, vp, vp, vp, i]
        _lib.oracle_projection_flips.argtypes = [C.POINTER(_Rig), vp, C.POINTER(_Grid), i, i, i]
        _lib.oracle_projection_flips.restype = i64
        _lib.oracle_max_threads.restype = i
        _lib.oracle_surface.argtypes = [vp, C.POINTER(_Grid), i, i, vp, i64]
        _lib.oracle_surface.restype = i64
        _lib.oracle_smooth_threshold.argtypes = [vp, C.POINTER(_Grid), d, vp, vp]
        _lib.oracle_color.argtypes = [C.POINTER(_Rig), C.POINTER(_Grid), vp, vp, vp, d, d, i64,
                                      vp, vp, vp, vp]
        _lib.oracle_train_background.argtypes = [i, i64, vp, d, vp, vp]
        _lib.oracle_train_background_elems.argtypes = [i, i64, vp, d, vp, vp]
        _lib.oracle_pixel_nch.argtypes = [i, vp, vp, vp, d, d, vp, vp, vp]
        _lib.oracle_slm_image_nch.argtypes = [i, i64, vp, vp, vp, d, d, vp, vp, vp, i]
        _lib.oracle_project_pinned_uv.argtypes = [vp, i, i, i, i, i, vp, vp]
        _lib.oracle_project_pinned_uv.restype = i
        _lib.oracle_bilinear.argtypes = [vp, i, i, d, d]
        _lib.oracle_bilinear.restype = d
        _lib.oracle_fuse_bilinear.argtypes = [C.POINTER(_Rig), C.POINTER(_Grid), vp, d, d, i, i,
                                              vp, vp, vp, i]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def max_threads() -> int:
    return int(lib().oracle_max_threads())


# ---------------------------------------------------------------- stage 1

def view_likelihood(slm: float, p_occ: float = 0.5):
    """(ln P(S|V=1), ln P(S|V=0)) for a hand-set SLM value, Eq (5)-(9)."""
    a, b = C.c_double(), C.c_double()
    lib().oracle_view_likelihood(float(slm), float(p_occ), C.byref(a), C.byref(b))
    return a.value, b.value


def slm_image(img, mu, sigma, sigma_floor=1.0, p_occ=0.5, nthreads=1):
    """Per-pixel SLM (Eq 1-2) and per-view log-likelihoods (Eq 5-9).

    img uint8 [..., nch]; mu, sigma float32 [..., nch] (same leading shape);
    nch = 3 (RGB, oracle_slm_image) or any other channel count, e.g. 1 for
    grayscale (oracle_slm_image_nch, U = 256^-nch; NEXT-3, R#25).
    Returns (slm, lnp1, lnp0) float64 arrays of the leading shape."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    mu = np.ascontiguousarray(mu, dtype=np.float32)
    sigma = np.ascontiguousarray(sigma, dtype=np.float32)
    shape = img.shape[:-1]
    nch = img.shape[-1]
    n = int(np.prod(shape)) if shape else 1
    assert mu.shape == img.shape and sigma.shape == img.shape
    slm = np.empty(n, np.float64)
    l1 = np.empty(n, np.float64)
    l0 = np.empty(n, np.float64)
    if nch == 3:
        lib().oracle_slm_image(n, 1, _p(img), _p(mu), _p(sigma), float(sigma_floor), float(p_occ),
                               _p(slm), _p(l1), _p(l0), int(nthreads))
    else:
        lib().oracle_slm_image_nch(int(nch), n, _p(img), _p(mu), _p(sigma), float(sigma_floor),
                                   float(p_occ), _p(slm), _p(l1), _p(l0), int(nthreads))
    return slm.reshape(shape), l1.reshape(shape), l0.reshape(shape)


def pixel_nch(I, mu, sigma, sigma_floor=1.0, p_occ=0.5):
    """One pixel of any channel count (oracle_pixel_nch): (slm, lnp1, lnp0)."""
    I = np.ascontiguousarray(np.asarray(I, np.uint8).reshape(-1))
    mu = np.ascontiguousarray(np.asarray(mu, np.float32).reshape(-1))
    sigma = np.ascontiguousarray(np.asarray(sigma, np.float32).reshape(-1))
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    lib().oracle_pixel_nch(int(I.size), _p(I), _p(mu), _p(sigma), float(sigma_floor), float(p_occ),
                           C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


# ---------------------------------------------------------------- projection

def precompose(P, origin, spacing) -> np.ndarray:
    """O4: A = S P T rounded to float, per camera. P: [ncam, 3, 4] float64."""
    P = np.ascontiguousarray(np.asarray(P, np.float64).reshape(-1, 12))
    org = np.ascontiguousarray(np.asarray(origin, np.float64))
    A = np.empty((P.shape[0], 12), np.float32)
    for c in range(P.shape[0]):
        lib().oracle_precompose(_p(P[c]), _p(org), float(spacing), _p(A[c]))
    return A


def project_pinned(A, W, H, ijk) -> np.ndarray:
    """O5 for many lattice points: returns int32 [n, 3] = (inview, px, py)."""
    A = np.ascontiguousarray(np.asarray(A, np.float32).reshape(12))
    ijk = np.ascontiguousarray(np.asarray(ijk, np.int32).reshape(-1, 3))
    out = np.empty_like(ijk)
    lib().oracle_project_pinned_batch(_p(A), int(W), int(H), ijk.shape[0], _p(ijk), _p(out))
    return out


def project_pinned_uv(A, W, H, i, j, k):
    """The pinned projection's float (u, v) (the +1/2 folded in) and the in-view
    decision; (0, nan, nan) when out of view (NEXT-3 bilinear, R#26)."""
    A = np.ascontiguousarray(np.asarray(A, np.float32).reshape(12))
    u, v = C.c_float(np.nan), C.c_float(np.nan)
    r = lib().oracle_project_pinned_uv(_p(A), int(W), int(H), int(i), int(j), int(k),
                                       C.byref(u), C.byref(v))
    return r, u.value, v.value


def bilinear(img, x, y):
    """oracle_bilinear: bilinear sample of a 2-D float64 image at the continuous
    pixel position (x, y), neighbours clamped to the image."""
    img = np.ascontiguousarray(np.asarray(img, np.float64))
    H, W = img.shape
    return float(lib().oracle_bilinear(_p(img), int(W), int(H), float(x), float(y)))


def project_exact(P, origin, spacing, W, H, i, j, k):
    P = np.ascontiguousarray(np.asarray(P, np.float64).reshape(12))
    org = np.ascontiguousarray(np.asarray(origin, np.float64))
    px, py = C.c_int(-1), C.c_int(-1)
    r = lib().oracle_project_exact(_p(P), _p(org), float(spacing), int(W), int(H), int(i),
                                   int(j), int(k), C.byref(px), C.byref(py))
    return r, px.value, py.value


# ---------------------------------------------------------------- stage 2

def _grid(g) -> _Grid:
    o = (C.c_double * 3)(*[float(x) for x in g.origin])
    return _Grid(o, float(g.spacing), int(g.xlen), int(g.ylen), int(g.zlen))


class _RigHolder:
    def __init__(self, A, W, H, p_occ):
        self.A = np.ascontiguousarray(A, np.float32)
        self.W = np.ascontiguousarray(W, np.int32)
        self.H = np.ascontiguousarray(H, np.int32)
        self.rig = _Rig(len(self.W), self.A.ctypes.data, self.W.ctypes.data,
                        self.H.ctypes.data, float(p_occ))


def _ptrs(arrs):
    return np.array([a.ctypes.data for a in arrs], dtype=np.uint64)


def reconstruct(P, W, H, grid, frames, mu, sigma, sigma_floor=1.0, p_occ=0.5, p_vox=0.5,
                tau=0.5, k0=0, k1=None, nthreads=1, want_slm=False, sampling="nearest"):
    """Whole-grid oracle: Eq (1)-(9) per pixel, Eq (3)-(4) per voxel, threshold.

    frames / mu / sigma: per camera [H, W, nch] (uint8 / float32 / float32),
    nch = 3 (RGB) or 1 (grayscale, NEXT-3).  sampling: "nearest" (R#10, the
    hot path) or "bilinear" (NEXT-3, R#26: oracle_fuse_bilinear on the
    SLM images).
    Returns dict(L=float64 [nvox_slab], post=float64, bits=uint32 words of the
    slab [k0,k1), lnp1/lnp0 per camera, A=the pre-composed matrices)."""
    k1 = grid.zlen if k1 is None else k1
    ncam = len(W)
    A = precompose(P, grid.origin, grid.spacing)
    l1s, l0s, slms = [], [], []
    for c in range(ncam):
        s, l1, l0 = slm_image(frames[c], mu[c], sigma[c], sigma_floor, p_occ, nthreads)
        l1s.append(np.ascontiguousarray(l1.reshape(-1)))
        l0s.append(np.ascontiguousarray(l0.reshape(-1)))
        slms.append(s)
    rh = _RigHolder(A, W, H, p_occ)
    g = _grid(grid)
    n = grid.xlen * grid.ylen * (k1 - k0)
    L = np.empty(n, np.float64)
    post = np.empty(n, np.float64)
    bits = np.zeros((n + 31) // 32, np.uint32)
    if sampling == "bilinear":
        sl = [np.ascontiguousarray(x.reshape(-1), np.float64) for x in slms]
        lib().oracle_fuse_bilinear(C.byref(rh.rig), C.byref(g), _p(_ptrs(sl)), float(p_vox),
                                   float(tau), int(k0), int(k1), _p(L), _p(post), _p(bits),
                                   int(nthreads))
    elif sampling == "nearest":
        p1, p0 = _ptrs(l1s), _ptrs(l0s)
        lib().oracle_fuse(C.byref(rh.rig), C.byref(g), _p(p1), _p(p0), float(p_vox), float(tau),
                          int(k0), int(k1), _p(L), _p(post), _p(bits), int(nthreads))
    else:
        raise ValueError(sampling)
    out = dict(L=L, post=post, bits=bits, lnp1=l1s, lnp0=l0s, A=A)
    if want_slm:
        out["slm"] = slms
    return out


def fuse_views(P, W, H, grid, lnp1, lnp0, p_occ=0.5, p_vox=0.5, tau=0.5, k0=0, k1=None,
               nthreads=1):
    """Eq (3)-(4) + threshold from given per-camera ln P(S|V=1), ln P(S|V=0)
    images (e.g. built from hand-set SLM values with ``view_likelihood``)."""
    k1 = grid.zlen if k1 is None else k1
    A = precompose(P, grid.origin, grid.spacing)
    rh = _RigHolder(A, W, H, p_occ)
    g = _grid(grid)
    l1s = [np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1)) for a in lnp1]
    l0s = [np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1)) for a in lnp0]
    n = grid.xlen * grid.ylen * (k1 - k0)
    L = np.empty(n, np.float64)
    post = np.empty(n, np.float64)
    bits = np.zeros((n + 31) // 32, np.uint32)
    lib().oracle_fuse(C.byref(rh.rig), C.byref(g), _p(_ptrs(l1s)), _p(_ptrs(l0s)), float(p_vox),
                      float(tau), int(k0), int(k1), _p(L), _p(post), _p(bits), int(nthreads))
    return dict(L=L, post=post, bits=bits)


def fuse_bilinear_slm(P, W, H, grid, slm, p_occ=0.5, p_vox=0.5, tau=0.5, k0=0, k1=None,
                      nthreads=1):
    """NEXT-3 bilinear fusion (oracle_fuse_bilinear) from given per-camera SLM
    images (float64 [H, W], e.g. hand-set for the pins)."""
    k1 = grid.zlen if k1 is None else k1
    A = precompose(P, grid.origin, grid.spacing)
    rh = _RigHolder(A, W, H, p_occ)
    g = _grid(grid)
    sl = [np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1)) for a in slm]
    n = grid.xlen * grid.ylen * (k1 - k0)
    L = np.empty(n, np.float64)
    post = np.empty(n, np.float64)
    bits = np.zeros((n + 31) // 32, np.uint32)
    lib().oracle_fuse_bilinear(C.byref(rh.rig), C.byref(g), _p(_ptrs(sl)), float(p_vox),
                               float(tau), int(k0), int(k1), _p(L), _p(post), _p(bits),
                               int(nthreads))
    return dict(L=L, post=post, bits=bits)


def fuse_sample(P, W, H, grid, frames, mu, sigma, vox, sigma_floor=1.0, p_occ=0.5, p_vox=0.5,
                nthreads=1):
    """Oracle log-odds (and posterior) of the listed linear voxel indices only."""
    A = precompose(P, grid.origin, grid.spacing)
    rh = _RigHolder(A, W, H, p_occ)
    g = _grid(grid)
    fr = [np.ascontiguousarray(f, np.uint8) for f in frames]
    mu = [np.ascontiguousarray(m, np.float32) for m in mu]
    sg = [np.ascontiguousarray(s, np.float32) for s in sigma]
    vox = np.ascontiguousarray(np.asarray(vox, np.int64))
    L = np.empty(vox.shape[0], np.float64)
    post = np.empty(vox.shape[0], np.float64)
    lib().oracle_fuse_sample(C.byref(rh.rig), C.byref(g), _p(_ptrs(fr)), _p(_ptrs(mu)),
                             _p(_ptrs(sg)), float(sigma_floor), float(p_vox), vox.shape[0],
                             _p(vox), _p(L), _p(post), int(nthreads))
    return L, post


def color(P, W, H, grid, frames, mu, sigma, vox, slm_gate=0.5, sigma_floor=1.0, p_occ=0.5):
    """NEXT-4: per listed voxel, the mean
    8-bit RGB over the cameras whose pinned nearest pixel is in view and has
    SLM > slm_gate.  Returns (rgb float64 [n, 3] (0 where unset), count int32
    [n], margin float64 [n] = min |SLM - slm_gate| over the in-view cameras)."""
    A = precompose(P, grid.origin, grid.spacing)
    rh = _RigHolder(A, W, H, p_occ)
    g = _grid(grid)
    fr = [np.ascontiguousarray(f, np.uint8) for f in frames]
    mu = [np.ascontiguousarray(m, np.float32) for m in mu]
    sg = [np.ascontiguousarray(s, np.float32) for s in sigma]
    vox = np.ascontiguousarray(np.asarray(vox, np.int64))
    n = vox.shape[0]
    rgb = np.empty((n, 3), np.float64)
    cnt = np.empty(n, np.int32)
    margin = np.empty(n, np.float64)
    lib().oracle_color(C.byref(rh.rig), C.byref(g), _p(_ptrs(fr)), _p(_ptrs(mu)), _p(_ptrs(sg)),
                       float(sigma_floor), float(slm_gate), n, _p(vox), _p(rgb), _p(cnt),
                       _p(margin))
    return rgb, cnt, margin


def train_background(frames, sigma_floor=1.0):
    """NEXT-3: per-pixel, per-channel mean and population standard
    deviation of a list of [H, W, nch] uint8 frames (nch = 3 RGB, 1 grayscale),
    sigma clamped to the floor.  Returns (mean, sigma) float64 [H, W, nch]."""
    fr = [np.ascontiguousarray(f, np.uint8) for f in frames]
    if not fr:
        raise ValueError("EmptyInput")
    if any(f.shape != fr[0].shape for f in fr):
        raise ValueError("DimensionMismatch")
    mean = np.empty(fr[0].shape, np.float64)
    sd = np.empty(fr[0].shape, np.float64)
    if fr[0].shape[-1] == 3:
        lib().oracle_train_background(len(fr), fr[0].size // 3, _p(_ptrs(fr)), float(sigma_floor),
                                      _p(mean), _p(sd))
    else:
        lib().oracle_train_background_elems(len(fr), fr[0].size, _p(_ptrs(fr)), float(sigma_floor),
                                            _p(mean), _p(sd))
    return mean, sd


def projection_flips(P, W, H, grid, k0=0, k1=None, p_occ=0.5, nthreads=1) -> int:
    """Diagnostic (i): voxel-camera pairs whose pinned FP32 pixel differs from
    the exact double nearest pixel."""
    k1 = grid.zlen if k1 is None else k1
    P = np.ascontiguousarray(np.asarray(P, np.float64).reshape(-1, 12))
    A = precompose(P, grid.origin, grid.spacing)
    rh = _RigHolder(A, W, H, p_occ)
    g = _grid(grid)
    return int(lib().oracle_projection_flips(C.byref(rh.rig), _p(P), C.byref(g), int(k0),
                                             int(k1), int(nthreads)))


def surface(bits, grid, k0=0, k1=None):
    """NEXT-2: linear indices (ascending) of the
    occupied voxels of slices [k0,k1) with at least one unoccupied 6-neighbour;
    outside the volume counts as unoccupied.  bits: uint32 words of the full grid."""
    k1 = grid.zlen if k1 is None else k1
    b = np.ascontiguousarray(np.asarray(bits).view(np.uint32))
    g = _grid(grid)
    n = int(lib().oracle_surface(_p(b), C.byref(g), int(k0), int(k1), None, 0))
    out = np.empty(max(n, 1), np.int64)
    lib().oracle_surface(_p(b), C.byref(g), int(k0), int(k1), _p(out), n)
    return out[:n]


def smooth_threshold(post, grid, tau=0.5):
    """NEXT-1: 3x3x3 zero-padded box average
    of the posterior (float64 [nvox], x-fastest), then occupied := smoothed > tau.
    Returns (smoothed float64 [nvox], bits uint32 words)."""
    post = np.ascontiguousarray(np.asarray(post, np.float64).reshape(-1))
    g = _grid(grid)
    sm = np.empty_like(post)
    bits = np.zeros((post.size + 31) // 32, np.uint32)
    lib().oracle_smooth_threshold(_p(post), C.byref(g), float(tau), _p(sm), _p(bits))
    return sm, bits


def scene_reconstruct(scene, frames, **kw):
    """Convenience: run ``reconstruct`` on a synth.Scene and a frame set."""
    return reconstruct(scene.P, scene.widths, scene.heights, scene.grid, frames, scene.mu,
                       scene.sigma, **kw)
