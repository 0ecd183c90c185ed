"""Synthetic PSFS scenes: ring camera rigs, Gaussian backgrounds, ray-cast bodies.

Recipe (SURVEY.md §8(d) "Synthetic inputs"):

* world in mm, z up; the volume of interest is the 2 m cube
  origin (-1000, -1000, 0), edge 2000 mm, at xlen=ylen=zlen = 32/128/256/512/1024
  (the paper's VOI is "xlen ... ylen ... zlen" samples);
* cameras on rings of radius 4000 mm looking at (0, 0, 1000); pinhole
  P = K [R | t], focal f = 0.5 H / tan(26 deg) so the cube's
  bounding sphere is inside every view, principal point ((W-1)/2, (H-1)/2)
  (integer pixel centres);
* background model per pixel per channel: mu a smooth random field in
  [20, 235], sigma uniform in [2, 8] (single Gaussian);
* background pixels: clamp(round(mu + sigma N(0,1))), the paper's
  single-Gaussian assumption; foreground (the ray hits the body) pixels:
  clamp(round(part colour + 6 N(0,1))) -- no contrast is enforced, so the
  likelihood maps get realistic holes;
* bodies: an ellipsoid, or the 10-cylinder body of Table 1
  in a walking / arm-waving motion for sequences.

Every random draw comes from numpy's counter-based Philox generator keyed by
(seed, stream id), so any frame of any camera can be regenerated on its own.
Nothing here evaluates a likelihood, a posterior or a voxel-to-pixel rounding:
those belong to the method and live only in ``oracle/`` and in the CUDA path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# geometry containers
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Grid:
    """Volume of interest: voxel (i,j,k) centre is
    origin + spacing * (idx + 0.5); x-fastest linear order."""

    origin: tuple
    spacing: float
    xlen: int
    ylen: int
    zlen: int

    @property
    def nvox(self) -> int:
        return self.xlen * self.ylen * self.zlen

    @property
    def nwords(self) -> int:
        return (self.nvox + 31) // 32


@dataclass
class Camera:
    """Calibrated pinhole view: P (3x4, world mm -> homogeneous px), W, H."""

    P: np.ndarray
    width: int
    height: int
    center: np.ndarray
    R: np.ndarray
    K: np.ndarray


@dataclass
class Scene:
    name: str
    grid: Grid
    cameras: list
    mu: np.ndarray      # float32 [ncam, H, W, nch] (nch = 3 RGB, 1 grayscale)
    sigma: np.ndarray   # float32 [ncam, H, W, nch]
    seed: int
    body: str = "skeleton"
    fg_noise: float = 6.0
    meta: dict = field(default_factory=dict)

    @property
    def ncam(self) -> int:
        return len(self.cameras)

    @property
    def channels(self) -> int:
        return int(self.mu.shape[-1])

    @property
    def P(self) -> np.ndarray:
        return np.stack([c.P for c in self.cameras]).astype(np.float64)

    @property
    def widths(self) -> np.ndarray:
        return np.array([c.width for c in self.cameras], dtype=np.int32)

    @property
    def heights(self) -> np.ndarray:
        return np.array([c.height for c in self.cameras], dtype=np.int32)


CUBE_ORIGIN = (-1000.0, -1000.0, 0.0)
CUBE_EDGE = 2000.0

# BASELINE.json configs[0..4]
CONFIGS = {
    "C1": dict(n=32, rings=[(4, 1000.0, 0.0)], W=64, H=48, frames=1,
               desc="32^3 grid, 4 cameras at 64x48, single synthetic frame"),
    "C2": dict(n=128, rings=[(8, 1000.0, 0.0)], W=640, H=480, frames=1,
               desc="128^3 grid, 8 cameras at 640x480, single frame"),
    "C3": dict(n=256, rings=[(8, 1000.0, 0.0)], W=1280, H=960, frames=300,
               desc="256^3 grid, 8 cameras at 1280x960, 300-frame sequence"),
    "C4": dict(n=512, rings=[(8, 600.0, 0.0), (8, 1600.0, 22.5)], W=1920, H=1080,
               frames=1, desc="512^3 grid, 16 cameras at 1920x1080"),
    "C5": dict(n=1024, rings=[(8, 300.0, 0.0), (8, 800.0, 11.25), (8, 1300.0, 22.5),
                             (8, 1800.0, 33.75)], W=1920, H=1080, frames=64,
               desc="1024^3 grid, 32 cameras at 1920x1080, frame-batched sequence"),
}

RING_RADIUS = 4000.0
LOOK_AT = np.array([0.0, 0.0, 1000.0])
HALF_FOV_V_DEG = 26.0


def config_seed(name: str) -> int:
    """seed = 1311*100 + config index."""
    return 1311 * 100 + int(name[1:])


def cube_grid(n: int) -> Grid:
    return Grid(CUBE_ORIGIN, CUBE_EDGE / n, n, n, n)


# --------------------------------------------------------------------------
# cameras
# --------------------------------------------------------------------------


def look_at_camera(center, target, W, H, f=None) -> Camera:
    """P = K [R | t] with x right, y down, z forward."""
    center = np.asarray(center, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    if f is None:
        f = 0.5 * H / math.tan(math.radians(HALF_FOV_V_DEG))
    zc = target - center
    zc /= np.linalg.norm(zc)
    up = np.array([0.0, 0.0, 1.0])
    xc = np.cross(zc, up)
    xc /= np.linalg.norm(xc)
    yc = np.cross(zc, xc)
    R = np.stack([xc, yc, zc])
    t = -R @ center
    K = np.array([[f, 0.0, (W - 1) / 2.0], [0.0, f, (H - 1) / 2.0], [0.0, 0.0, 1.0]])
    P = K @ np.concatenate([R, t[:, None]], axis=1)
    return Camera(P=P, width=int(W), height=int(H), center=center, R=R, K=K)


def ring_rig(rings, W, H, radius=RING_RADIUS, target=LOOK_AT):
    """Cameras equally spaced on horizontal rings.

    rings: list of (count, height_mm, azimuth_offset_deg)."""
    cams = []
    for count, height, off in rings:
        for c in range(count):
            az = math.radians(off + 360.0 * c / count)
            centre = (radius * math.cos(az), radius * math.sin(az), height)
            cams.append(look_at_camera(centre, target, W, H))
    return cams


# --------------------------------------------------------------------------
# background model
# --------------------------------------------------------------------------


def _rng(seed: int, *stream) -> np.random.Generator:
    key = [int(seed) & 0xFFFFFFFFFFFFFFFF]
    k2 = 0
    for s in stream:
        k2 = (k2 * 1000003 + int(s)) & 0xFFFFFFFFFFFFFFFF
    return np.random.Generator(np.random.Philox(key=np.array(key + [k2], dtype=np.uint64)))


def make_background(seed, cam, W, H, sigma_range=(2.0, 8.0), integer_mu=False,
                    const_sigma=None, channels=3):
    """mu: smooth random field in [20, 235]; sigma: uniform in sigma_range.
    channels: 3 (RGB) or 1 (grayscale, NEXT-3)."""
    rng = _rng(seed, 1, cam)
    y, x = np.mgrid[0:H, 0:W].astype(np.float32)
    mu = np.empty((H, W, channels), np.float32)
    for ch in range(channels):
        a = rng.uniform(0.5, 2.5, size=4)
        ph = rng.uniform(0, 2 * np.pi, size=4)
        field_ = (60.0 * np.sin(2 * np.pi * (a[0] * x / W + a[1] * y / H) + ph[0])
                  + 35.0 * np.sin(2 * np.pi * (a[2] * x / W - a[3] * y / H) + ph[1]))
        field_ += rng.uniform(-15.0, 15.0, size=(H, W)).astype(np.float32)
        mu[..., ch] = np.clip(127.5 + field_, 20.0, 235.0)
    if integer_mu:
        mu = np.round(mu).astype(np.float32)
    if const_sigma is not None:
        sigma = np.full((H, W, channels), const_sigma, np.float32)
    else:
        sigma = rng.uniform(sigma_range[0], sigma_range[1], size=(H, W, channels)).astype(np.float32)
    return mu, sigma


# --------------------------------------------------------------------------
# bodies (exact ray casting)
# --------------------------------------------------------------------------

PALETTE = np.array([
    [200, 40, 40], [40, 160, 60], [40, 60, 200], [220, 200, 40], [160, 40, 200],
    [40, 200, 200], [240, 120, 30], [120, 80, 40], [250, 250, 250], [10, 10, 10],
    [230, 150, 170],
], dtype=np.float32)


def ellipsoid_part(center=(0.0, 0.0, 1000.0), axes=(250.0, 180.0, 850.0)):
    return ("ellipsoid", np.asarray(center, float), np.asarray(axes, float))


def skeleton_parts(t: float = 0.0, walk: bool = False, wave: bool = False,
                   jitter: float = 0.0):
    """The 10 cylinders of Table 1 posed at time t (s).

    walk: x translation, triangle wave within +-600 mm at 1 m/s;
    wave: shoulder angle A sin(2 pi f t), A = 0.6 rad, f = 0.5 Hz.
    jitter: extra small deterministic pose offset (radians) for distinct frames."""
    x0 = 0.0
    if walk:
        period = 2.4  # 1.2 m there and back at 1 m/s
        ph = (t % period) / period
        x0 = -600.0 + 1200.0 * (2 * ph if ph < 0.5 else 2 - 2 * ph)
    arm = 0.6 * math.sin(2 * math.pi * 0.5 * t) if wave else 0.0
    arm += jitter
    leg = 0.35 * math.sin(2 * math.pi * 1.0 * t) if walk else 0.0
    leg += 0.5 * jitter

    def rot_y(v, ang):  # rotate (dx, dy, dz) about the y axis (swing in x-z)
        c, s = math.cos(ang), math.sin(ang)
        return np.array([c * v[0] + s * v[2], v[1], -s * v[0] + c * v[2]])

    def seg(p0, vec, r):
        p0 = np.asarray(p0, float) + np.array([x0, 0, 0])
        return ("cylinder", p0, p0 + vec, float(r))

    parts = []
    parts.append(seg((0, 0, 900), np.array([0, 0, 550.0]), 160))            # 1 torso
    for side, sgn in (("L", 1.0), ("R", -1.0)):                           # 2-5 legs
        swing = leg * sgn
        thigh = rot_y(np.array([0, 0, -420.0]), swing)
        parts.append(seg((0, 100 * sgn, 900), thigh, 75))
        knee = np.array([0, 100 * sgn, 900]) + thigh
        parts.append(seg(knee, rot_y(np.array([0, 0, -420.0]), swing * 0.5), 55))
    for side, sgn in (("L", 1.0), ("R", -1.0)):                           # 6-9 arms
        ang = arm * sgn
        upper = np.array([0.0, 300.0 * sgn * math.sin(abs(ang)), -300.0 * math.cos(ang)])
        parts.append(seg((0, 215 * sgn, 1420), upper, 50))
        elbow = np.array([0, 215 * sgn, 1420]) + upper
        parts.append(seg(elbow, upper * (260.0 / 300.0), 40))
    parts.append(seg((0, 0, 1500), np.array([0, 0, 220.0]), 95))           # 10 head
    return parts


def _ray_dirs(cam: Camera):
    H, W = cam.height, cam.width
    v, u = np.mgrid[0:H, 0:W]
    pix = np.stack([u.ravel(), v.ravel(), np.ones(H * W)], axis=0).astype(np.float64)
    d = cam.R.T @ (np.linalg.inv(cam.K) @ pix)
    return d.T  # [N, 3], pixel centres at integer coordinates


def _hit_ellipsoid(o, d, center, axes):
    o2 = (o - center) / axes
    d2 = d / axes
    A = np.einsum("ij,ij->i", d2, d2)
    B = 2.0 * (d2 @ o2)
    C = o2 @ o2 - 1.0
    disc = B * B - 4 * A * C
    ok = disc >= 0
    sq = np.sqrt(np.where(ok, disc, 0.0))
    t0 = (-B - sq) / (2 * A)
    t1 = (-B + sq) / (2 * A)
    t = np.where(t0 > 0, t0, t1)
    hit = ok & (t1 > 0)
    return hit, np.where(hit, t, np.inf)


def _hit_cylinder(o, d, p0, p1, r):
    axis = p1 - p0
    L = np.linalg.norm(axis)
    a = axis / L
    w = o - p0
    da = d @ a
    wa = w @ a
    dp = d - da[:, None] * a
    wp = w - wa * a
    A = np.einsum("ij,ij->i", dp, dp)
    B = 2.0 * (dp @ wp)
    C = wp @ wp - r * r
    disc = B * B - 4 * A * C
    eps = 1e-12
    par = A < eps
    sq = np.sqrt(np.maximum(disc, 0.0))
    Asafe = np.where(par, 1.0, A)
    tr0 = np.where(par, np.where(C <= 0, -np.inf, np.inf), (-B - sq) / (2 * Asafe))
    tr1 = np.where(par, np.where(C <= 0, np.inf, -np.inf), (-B + sq) / (2 * Asafe))
    tr_ok = par | (disc >= 0)
    dsafe = np.where(np.abs(da) < eps, 1.0, da)
    ta = (0.0 - wa) / dsafe
    tb = (L - wa) / dsafe
    inside_ax = (wa >= 0) & (wa <= L)
    ta0 = np.where(np.abs(da) < eps, np.where(inside_ax, -np.inf, np.inf), np.minimum(ta, tb))
    ta1 = np.where(np.abs(da) < eps, np.where(inside_ax, np.inf, -np.inf), np.maximum(ta, tb))
    enter = np.maximum(np.maximum(tr0, ta0), 0.0)
    exit_ = np.minimum(tr1, ta1)
    hit = tr_ok & (enter <= exit_)
    return hit, np.where(hit, enter, np.inf)


def _part_bbox(cam: Camera, part):
    """Pixel bounding box (r0, r1, c0, c1) of a part from its axis-aligned
    bounding box corners; None if some corner is not in front of the camera."""
    if part[0] == "ellipsoid":
        lo, hi = part[1] - part[2], part[1] + part[2]
    else:
        lo = np.minimum(part[1], part[2]) - part[3]
        hi = np.maximum(part[1], part[2]) + part[3]
    corners = np.array([[lo[0] if a else hi[0], lo[1] if b else hi[1], lo[2] if c else hi[2], 1.0]
                        for a in (0, 1) for b in (0, 1) for c in (0, 1)])
    x = corners @ cam.P.T
    if (x[:, 2] <= 1e-6).any():
        return None
    u, v = x[:, 0] / x[:, 2], x[:, 1] / x[:, 2]
    c0 = max(0, int(np.floor(u.min())) - 1)
    c1 = min(cam.width, int(np.ceil(u.max())) + 2)
    r0 = max(0, int(np.floor(v.min())) - 1)
    r1 = min(cam.height, int(np.ceil(v.max())) + 2)
    return r0, r1, c0, c1


def render_labels(cam: Camera, parts) -> np.ndarray:
    """Per-pixel index of the nearest body part hit by the pixel-centre ray
    (exact ray-quadric / ray-capped-cylinder test); -1 = none.
    Rays are only cast inside each part's projected bounding box (the part's
    convex AABB projects inside the hull of its projected corners)."""
    d_all = _ray_dirs(cam).reshape(cam.height, cam.width, 3)
    o = cam.center
    best_t = np.full((cam.height, cam.width), np.inf)
    label = np.full((cam.height, cam.width), -1, np.int16)
    for idx, part in enumerate(parts):
        bb = _part_bbox(cam, part)
        r0, r1, c0, c1 = bb if bb is not None else (0, cam.height, 0, cam.width)
        if r1 <= r0 or c1 <= c0:
            continue
        d = d_all[r0:r1, c0:c1].reshape(-1, 3)
        if part[0] == "ellipsoid":
            hit, t = _hit_ellipsoid(o, d, part[1], part[2])
        else:
            hit, t = _hit_cylinder(o, d, part[1], part[2], part[3])
        hit = hit.reshape(r1 - r0, c1 - c0)
        t = t.reshape(r1 - r0, c1 - c0)
        bt = best_t[r0:r1, c0:c1]
        closer = hit & (t < bt)
        best_t[r0:r1, c0:c1] = np.where(closer, t, bt)
        label[r0:r1, c0:c1] = np.where(closer, idx, label[r0:r1, c0:c1])
    return label


def render_silhouette(cam: Camera, parts) -> np.ndarray:
    """True binary silhouette (noise-free), bool [H, W]."""
    return render_labels(cam, parts) >= 0


def _noisy_frame(seed, frame, cam_idx, mu, sigma, labels, fg_noise):
    rng = _rng(seed, 2, frame, cam_idx)
    H, W, nch = mu.shape
    n_bg = rng.standard_normal((H, W, nch), dtype=np.float32)
    img = mu + sigma * n_bg
    fg = labels >= 0
    if fg.any():
        n_fg = rng.standard_normal((int(fg.sum()), nch), dtype=np.float32)
        cols = PALETTE[labels[fg] % len(PALETTE)]
        if nch != 3:  # grayscale: the palette colour's channel mean
            cols = cols.mean(axis=1, keepdims=True)
        img[fg] = cols + fg_noise * n_fg
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def _clean_frame(mu, labels):
    """Noise-free variant for the SFS limit: background I = mu exactly (mu must
    be integer-valued), foreground 80 grey levels away from mu in every channel."""
    img = mu.copy()
    fg = labels >= 0
    m = mu[fg]
    img[fg] = np.where(m < 128.0, m + 80.0, m - 80.0)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def body_parts(body: str, frame: int, fps: float = 30.0, motion: bool = False):
    t = frame / fps
    if body == "ellipsoid":
        return [ellipsoid_part()]
    if body == "skeleton":
        if motion:
            return skeleton_parts(t, walk=True, wave=True)
        # distinct frames without a sequence: deterministic small pose jitter
        return skeleton_parts(0.0, jitter=0.05 * ((frame * 7) % 11) / 10.0)
    if body == "both":
        return [ellipsoid_part(center=(450.0, 0.0, 1000.0), axes=(200, 150, 700))] + \
            skeleton_parts(0.0, jitter=0.05 * ((frame * 7) % 11) / 10.0)
    if body == "empty":
        return []
    raise ValueError(body)


def make_frames(scene: Scene, frame: int, mode: str = "noisy", motion: bool = False,
                labels_out: list | None = None) -> np.ndarray:
    """uint8 [ncam, H, W, nch] frame set for one time step (RGB or grayscale)."""
    parts = body_parts(scene.body, frame, motion=motion)
    out = []
    for c, cam in enumerate(scene.cameras):
        labels = render_labels(cam, parts) if parts else \
            np.full((cam.height, cam.width), -1, np.int16)
        if labels_out is not None:
            labels_out.append(labels)
        if mode == "noisy":
            out.append(_noisy_frame(scene.seed, frame, c, scene.mu[c], scene.sigma[c],
                                    labels, scene.fg_noise))
        elif mode == "clean":
            out.append(_clean_frame(scene.mu[c], labels))
        elif mode == "background":
            out.append(np.clip(np.rint(scene.mu[c]), 0, 255).astype(np.uint8))
        else:
            raise ValueError(mode)
    return np.stack(out)


def make_scene(name: str = "C1", body: str = "skeleton", seed: int | None = None,
               grid: Grid | None = None, integer_mu: bool = False, const_sigma=None,
               rings=None, W=None, H=None, channels: int = 3) -> Scene:
    """channels: 3 (8-bit RGB, the default) or 1 (8-bit grayscale, NEXT-3):
    mu / sigma / frames carry that many channels in their last axis."""
    cfg = CONFIGS[name]
    seed = config_seed(name) if seed is None else seed
    grid = grid or cube_grid(cfg["n"])
    W = W or cfg["W"]
    H = H or cfg["H"]
    cams = ring_rig(rings or cfg["rings"], W, H)
    mus, sigs = [], []
    for c, cam in enumerate(cams):
        mu, sg = make_background(seed, c, cam.width, cam.height, integer_mu=integer_mu,
                                 const_sigma=const_sigma, channels=channels)
        mus.append(mu)
        sigs.append(sg)
    return Scene(name=name, grid=grid, cameras=cams, mu=np.stack(mus), sigma=np.stack(sigs),
                 seed=seed, body=body, meta=dict(desc=cfg["desc"]))
