"""Seeded synthetic workloads standing in for BASELINE.json configs[0..4].

There is no public dataset for this path; every
array here is generated from ``np.random.default_rng(seed)`` so the CUDA
path, the CPU oracle and the reference all see identical inputs:

* body      union of 7 ellipsoids (torso, head, 4 legs, tail) in [-1, 1]^3,
            a cell kept where |approximate SDF at its centre| <= shell*cell;
            a per-config scale calibrates the leaf count (~30 k / ~1 M / ~4 M)
* FLUT      features N(0, 0.5) and density softplus(N(0, 1)), both rounded
            to fp32 (D8) in the reference column order h*C + c, density last
* rig       24 (or 32) joints along the ellipsoid axes, parents first;
            skin weights = softmax(beta / distance) over the 4 nearest joints,
            K = 4 slots sorted by joint index, fp64 (D5, D10)
* poses     axis-angle per joint (|theta| <= 0.3) converted to the
            reference's intrinsic XYZ Euler angles (D6); sinusoid walk (C3)
            and random walk (C4) sequences
* cameras   orbit cameras with focal = (W/2)/tan(20 deg) (D7), +z up

Seeds: geometry/features/rig use ``seed``; the pose of frame f uses
``seed + 1000 + f``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import kinematics as K

# (centre, radii) of the template body, probe P1.
_ELLIPSOIDS = (
    ((0.0, 0.0, 0.0), (0.45, 0.2, 0.2)),       # torso
    ((0.55, 0.0, 0.15), (0.15, 0.12, 0.12)),   # head
    ((0.3, 0.12, -0.3), (0.06, 0.06, 0.25)),   # legs
    ((0.3, -0.12, -0.3), (0.06, 0.06, 0.25)),
    ((-0.3, 0.12, -0.3), (0.06, 0.06, 0.25)),
    ((-0.3, -0.12, -0.3), (0.06, 0.06, 0.25)),
    ((-0.6, 0.0, 0.05), (0.2, 0.04, 0.04)),    # tail
)


def _template_joints(n_joints: int):
    """Joint positions along the ellipsoid axes and their parents."""
    pos = [(0.0, 0.0, 0.0)]                       # 0 root (torso centre)
    par = [-1]

    def add(p, parent):
        pos.append(p)
        par.append(parent)
        return len(pos) - 1

    # spine towards the head, neck, head
    a = add((0.15, 0.0, 0.0), 0)
    b = add((0.30, 0.0, 0.0), a)
    c = add((0.42, 0.0, 0.05), b)
    d = add((0.50, 0.0, 0.12), c)
    e = add((0.60, 0.0, 0.15), d)
    add((0.68, 0.0, 0.15), e)
    # spine towards the tail, tail
    f = add((-0.15, 0.0, 0.0), 0)
    g = add((-0.30, 0.0, 0.0), f)
    h = add((-0.42, 0.0, 0.03), g)
    i = add((-0.55, 0.0, 0.05), h)
    tail_tip = add((-0.70, 0.0, 0.05), i)
    leg_depth = 4 if n_joints >= 32 else 3
    for sx, hip_parent in ((0.3, b), (-0.3, g)):
        for sy in (0.12, -0.12):
            prev = hip_parent
            for z in (-0.1, -0.3, -0.5, -0.55)[:leg_depth]:
                prev = add((sx, sy, z), prev)
    if n_joints >= 32:
        t2 = add((-0.76, 0.0, 0.05), tail_tip)
        add((-0.80, 0.0, 0.05), t2)
        add((0.60, 0.06, 0.26), e)                # ears
        add((0.60, -0.06, 0.26), e)
    if len(pos) != n_joints:
        raise ValueError(f"template supports 24 or 32 joints, got {n_joints}")
    return np.array(pos, dtype=np.float64), np.array(par, dtype=np.int32)


def body_cells(resolution: int, shell: float, scale: float) -> np.ndarray:
    """(N, 3) int32 cells of the ellipsoid-union shell, x-major order."""
    n = resolution
    cell = 2.0 / n
    centres = [(np.array(c) * scale, np.array(r) * scale) for c, r in _ELLIPSOIDS]
    # bounding box of the union, padded by the shell
    pad = (shell + 1) * cell
    lo = np.min([c - r for c, r in centres], axis=0) - pad
    hi = np.max([c + r for c, r in centres], axis=0) + pad
    ilo = np.clip(np.floor((lo + 1.0) / cell).astype(int), 0, n - 1)
    ihi = np.clip(np.ceil((hi + 1.0) / cell).astype(int), 0, n - 1)
    ys = np.arange(ilo[1], ihi[1] + 1)
    zs = np.arange(ilo[2], ihi[2] + 1)
    py = -1.0 + (ys + 0.5) * cell
    pz = -1.0 + (zs + 0.5) * cell
    out = []
    thr = shell * cell
    for x in range(ilo[0], ihi[0] + 1):
        px = -1.0 + (x + 0.5) * cell
        sdf = np.full((ys.size, zs.size), np.inf)
        for c, r in centres:
            dx = (px - c[0]) / r[0]
            if abs(dx) > 1.0 + thr / r.min():
                continue
            dy = ((py - c[1]) / r[1])[:, None]
            dz = ((pz - c[2]) / r[2])[None, :]
            s = (np.sqrt(dx * dx + dy * dy + dz * dz) - 1.0) * r.min()
            np.minimum(sdf, s, out=sdf)
        yy, zz = np.nonzero(np.abs(sdf) <= thr)
        if yy.size:
            out.append(np.stack([np.full(yy.size, x), ys[yy], zs[zz]], axis=1))
    return np.concatenate(out).astype(np.int32)


def make_flut(n: int, degree: int, channels: int, rng: np.random.Generator,
              chunk: int = 1 << 18) -> np.ndarray:
    """(n, H*C+1) float32: N(0,0.5) coefficients, softplus(N(0,1)) density."""
    h = (degree + 1) * (degree + 1)
    w = h * channels + 1
    out = np.empty((n, w), dtype=np.float32)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        out[a:b, :-1] = rng.standard_normal((b - a, w - 1), dtype=np.float32) * np.float32(0.5)
    z = rng.standard_normal(n)
    out[:, -1] = np.logaddexp(0.0, z).astype(np.float32)
    return out


def skin_weights(centers: np.ndarray, joints: np.ndarray, k: int = 4, beta: float = 0.05,
                 chunk: int = 1 << 18):
    """Softmax over inverse distances to the k nearest joints; slots sorted
    by joint index; (N, k) int32 and (N, k) float64 summing to 1."""
    n = centers.shape[0]
    idx = np.empty((n, k), dtype=np.int32)
    wts = np.empty((n, k), dtype=np.float64)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        d = np.linalg.norm(centers[a:b, None, :] - joints[None, :, :], axis=2)
        near = np.argpartition(d, k - 1, axis=1)[:, :k]
        near.sort(axis=1)
        dn = np.take_along_axis(d, near, axis=1)
        logit = beta / np.maximum(dn, 1e-6)
        logit -= logit.max(axis=1, keepdims=True)
        e = np.exp(logit)
        idx[a:b] = near
        wts[a:b] = e / e.sum(axis=1, keepdims=True)
    return idx, wts


def axis_angle_euler(rng: np.random.Generator, n_joints: int, max_angle: float) -> np.ndarray:
    """Random axis and |angle| <= max_angle per joint, as XYZ Euler (D6)."""
    axes = rng.normal(size=(n_joints, 3))
    axes /= np.linalg.norm(axes, axis=1, keepdims=True)
    ang = rng.uniform(-max_angle, max_angle, size=n_joints)
    return np.stack([K.euler_xyz_from_quat(K.q_from_axis_angle(axes[j], ang[j]))
                     for j in range(n_joints)])


def _rotvec_euler(v: np.ndarray) -> np.ndarray:
    out = []
    for r in v:
        a = float(np.linalg.norm(r))
        out.append(K.euler_xyz_from_quat(K.q_from_axis_angle(r, a)) if a > 0 else np.zeros(3))
    return np.stack(out)


def sinusoid_sequence(seed: int, n_joints: int, frames: int, amp: float = 0.4):
    """C3: per-joint rotation vector = sum of 3 sinusoids, |component| <= amp."""
    rng = np.random.default_rng(seed + 1000)
    a = rng.uniform(0.0, amp / 3.0, size=(3, n_joints, 3))
    w = rng.uniform(0.05, 0.3, size=(3, n_joints, 3))
    ph = rng.uniform(0.0, 2 * np.pi, size=(3, n_joints, 3))
    seq = []
    for f in range(frames):
        v = (a * np.sin(w * f + ph)).sum(axis=0)
        seq.append(_rotvec_euler(v))
    return seq


def random_walk_sequence(seed: int, n_joints: int, frames: int, step: float = 0.05,
                         limit: float = 0.4):
    """C4: clipped Gaussian random walk of per-joint rotation vectors."""
    rng = np.random.default_rng(seed + 1000)
    v = np.zeros((n_joints, 3))
    seq = []
    for _ in range(frames):
        v = np.clip(v + rng.normal(scale=step, size=v.shape), -limit, limit)
        seq.append(_rotvec_euler(v))
    return seq


@dataclass
class Scene:
    """One synthetic character plus the frames/views a config renders."""

    name: str
    resolution: int
    lo: np.ndarray
    hi: np.ndarray
    cells: np.ndarray                 # (N, 3) int32 canonical cells
    flut32: np.ndarray                # (N, H*C+1) float32, density last
    degree: int
    channels: int
    rig: K.Rig
    skin_idx: np.ndarray              # (N, 4) int32
    skin_w: np.ndarray                # (N, 4) float64
    poses: list = field(default_factory=list)     # per frame: (J, 3) raw XYZ Euler (wrapped by PoseSpec)
    cameras: list = field(default_factory=list)   # per frame: list of PinholeCamera
    lambda_th: float = 1e-4
    sigma_dep: float = 5.0

    @property
    def n_voxels(self) -> int:
        return int(self.cells.shape[0])

    @property
    def cell_size(self) -> np.ndarray:
        return (self.hi - self.lo) / self.resolution

    def centers(self) -> np.ndarray:
        """VoxelSet.centers (volume.py:82-85) in the same op order."""
        return self.lo + (self.cells.astype(np.float64) + 0.5) * self.cell_size

    def flut64(self, rows=None) -> np.ndarray:
        """Exact fp64 widening of the fp32 FLUT (what the reference holds)."""
        src = self.flut32 if rows is None else self.flut32[rows]
        return src.astype(np.float64)

    def rays_per_frame(self) -> int:
        return sum(c.width * c.height for c in self.cameras[0])


# per-config body scale calibrated for the target leaf counts
_CONFIGS = {
    # name: (resolution, shell, scale, channels, joints, image (W,H), views, frames)
    "c0": dict(resolution=128, shell=3, scale=0.76, channels=16, joints=24,
               image=(256, 256)),
    "c1": dict(resolution=128, shell=3, scale=0.76, channels=16, joints=24,
               image=(512, 512)),
    "c2": dict(resolution=512, shell=4, scale=0.95, channels=32, joints=24,
               image=(1024, 1024)),
    "c3": dict(resolution=512, shell=4, scale=0.95, channels=32, joints=24,
               image=(1024, 1024)),
    "c4": dict(resolution=1024, shell=3, scale=1.1, channels=32, joints=32,
               image=(1440, 1600)),
}

CONFIG_NAMES = tuple(_CONFIGS)


def make_scene(name: str, *, seed: int = 0, frames: int | None = None,
               resolution: int | None = None, image=None, shell=None,
               scale=None, channels=None, with_flut: bool = True) -> Scene:
    """Build configs[k] (``name`` = "c0".."c4"). Keyword overrides shrink a
    config for parity tests while keeping its structure."""
    cfg = dict(_CONFIGS[name])
    if resolution is not None:
        cfg["resolution"] = resolution
    if image is not None:
        cfg["image"] = tuple(image)
    if shell is not None:
        cfg["shell"] = shell
    if scale is not None:
        cfg["scale"] = scale
    if channels is not None:
        cfg["channels"] = channels
    res = cfg["resolution"]
    rng = np.random.default_rng(seed)
    cells = body_cells(res, cfg["shell"], cfg["scale"])
    joints, parents = _template_joints(cfg["joints"])
    joints = joints * cfg["scale"]
    bind_t = joints.copy()
    bind_t[1:] = joints[1:] - joints[parents[1:]]
    rig = K.Rig(parents=parents, bind_q=np.tile([1.0, 0.0, 0.0, 0.0], (len(parents), 1)),
                bind_t=bind_t)
    lo = np.full(3, -1.0)
    hi = np.full(3, 1.0)
    centers = lo + (cells.astype(np.float64) + 0.5) * ((hi - lo) / res)
    canon = K.canonical_globals(rig)
    joint_pos = np.stack([t for _, t in canon])
    skin_idx, skin_w = skin_weights(centers, joint_pos)
    flut = make_flut(cells.shape[0], 2, cfg["channels"], rng) if with_flut else \
        np.zeros((cells.shape[0], 9 * cfg["channels"] + 1), dtype=np.float32)

    W, H = cfg["image"]
    focal = K.focal_for_fov(W, 40.0)
    el = math.radians(15.0)
    nj = cfg["joints"]
    poses: list = []
    cams: list = []
    if name in ("c0", "c2"):
        n_frames = frames or 1
        for f in range(n_frames):
            prng = np.random.default_rng(seed + 1000 + f)
            poses.append(axis_angle_euler(prng, nj, 0.3))
            cams.append([K.orbit(math.radians(45.0), el, 2.5, W, H, focal)])
    elif name == "c1":
        prng = np.random.default_rng(seed + 1000)
        poses.append(axis_angle_euler(prng, nj, 0.3))
        cams.append([K.orbit(math.radians(45.0 * k), el, 2.5, W, H, focal) for k in range(8)])
    elif name == "c3":
        n_frames = frames or 64
        poses = sinusoid_sequence(seed, nj, n_frames)
        cams = [[K.orbit(math.radians(45.0 + 5.6 * f), el, 2.5, W, H, focal)]
                for f in range(n_frames)]
    elif name == "c4":
        n_frames = frames or 48
        poses = random_walk_sequence(seed, nj, n_frames)
        jr = np.random.default_rng(seed + 2000)
        for _ in range(n_frames):
            az = math.radians(jr.uniform(-5.0, 5.0))
            e2 = math.radians(jr.uniform(-5.0, 5.0))
            head = K.orbit(az, e2, 2.0, W, H, focal)
            r, o = head.cam_to_world()
            right = r[:, 0]
            eyes = []
            for s in (-0.032, 0.032):
                pos = o + s * right
                eyes.append(K.look_at(pos, pos + r[:, 2], W, H, focal))
            cams.append(eyes)
    return Scene(name=name, resolution=res, lo=lo, hi=hi, cells=cells, flut32=flut,
                 degree=2, channels=cfg["channels"], rig=rig, skin_idx=skin_idx,
                 skin_w=skin_w, poses=poses, cameras=cams)
