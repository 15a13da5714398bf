"""Host-side rig and camera math that feeds the device path.

Forward kinematics runs on the host (J <= 64 joints, microseconds) exactly
as the reference does it, because the warp kernel's bit-exact Morton keys
depend on bit-identical per-joint delta matrices. Every formula below is a
restatement of the reference's numpy arithmetic in the same operation
order, so on any given host it produces the same doubles as:

* quaternion helpers   animvox/geometry.py:33-117
* RigidTransform       animvox/geometry.py:124-169 (compose/invert/matrix)
* Pose angle wrap      animvox/rigging.py:65-67, 94
* forward_kinematics   animvox/rigging.py:228-247
* per-joint deltas     animvox/rigging.py:343-347
* look_at/orbit camera animvox/synthetic.py:294-373
* camera-to-world      animvox/geometry.py:242-263 (rays_for_camera)

A rigid transform is a plain ``(q, t)`` tuple: unit quaternion (w, x, y, z)
then translation, y = R(q) x + t.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ContractViolation

_F64 = np.float64


# ---------------------------------------------------------------------------
# quaternions (w, x, y, z)


def qmul(a, b) -> np.ndarray:
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array(
        [
            aw * bw - ax * bx - ay * by - az * bz,
            aw * bx + ax * bw + ay * bz - az * by,
            aw * by - ax * bz + ay * bw + az * bx,
            aw * bz + ax * by - ay * bx + az * bw,
        ]
    )


def qconj(q) -> np.ndarray:
    return np.array([q[0], -q[1], -q[2], -q[3]])


def qnormalize(q) -> np.ndarray:
    q = np.asarray(q, dtype=_F64)
    n = np.linalg.norm(q)
    if n == 0.0:
        raise ContractViolation("zero quaternion")
    return q / n


def qmatrix(q) -> np.ndarray:
    """3x3 rotation matrix of a unit quaternion."""
    w, x, y, z = q
    return np.array(
        [
            [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
            [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
            [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
        ]
    )


def qrotate(q, v) -> np.ndarray:
    return qmatrix(q) @ np.asarray(v, dtype=_F64)


def q_from_axis_angle(axis, angle: float) -> np.ndarray:
    axis = np.asarray(axis, dtype=_F64)
    n = np.linalg.norm(axis)
    if n == 0.0:
        return np.array([1.0, 0.0, 0.0, 0.0])
    half = 0.5 * angle
    return np.concatenate([[math.cos(half)], math.sin(half) / n * axis])


def q_from_euler_xyz(angles) -> np.ndarray:
    """Intrinsic X then Y then Z: q = qz * qy * qx."""
    rx, ry, rz = (float(a) for a in angles)
    qx = q_from_axis_angle([1, 0, 0], rx)
    qy = q_from_axis_angle([0, 1, 0], ry)
    qz = q_from_axis_angle([0, 0, 1], rz)
    return qmul(qz, qmul(qy, qx))


def q_from_matrix(m) -> np.ndarray:
    """Shepperd's method, w >= 0, renormalised."""
    m = np.asarray(m, dtype=_F64)
    tr = np.trace(m)
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2
        q = np.array([0.25 * s, (m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s,
                      (m[1, 0] - m[0, 1]) / s])
    elif m[0, 0] >= m[1, 1] and m[0, 0] >= m[2, 2]:
        s = math.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2]) * 2
        q = np.array([(m[2, 1] - m[1, 2]) / s, 0.25 * s, (m[0, 1] + m[1, 0]) / s,
                      (m[0, 2] + m[2, 0]) / s])
    elif m[1, 1] >= m[2, 2]:
        s = math.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2]) * 2
        q = np.array([(m[0, 2] - m[2, 0]) / s, (m[0, 1] + m[1, 0]) / s, 0.25 * s,
                      (m[1, 2] + m[2, 1]) / s])
    else:
        s = math.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1]) * 2
        q = np.array([(m[1, 0] - m[0, 1]) / s, (m[0, 2] + m[2, 0]) / s,
                      (m[1, 2] + m[2, 1]) / s, 0.25 * s])
    if q[0] < 0:
        q = -q
    return qnormalize(q)


def euler_xyz_from_quat(q) -> np.ndarray:
    """Inverse of q_from_euler_xyz up to rounding (used only to express
    sampled axis-angle poses in the reference's Euler convention, D6)."""
    r = qmatrix(qnormalize(q))
    ry = math.asin(max(-1.0, min(1.0, -float(r[2, 0]))))
    rx = math.atan2(float(r[2, 1]), float(r[2, 2]))
    rz = math.atan2(float(r[1, 0]), float(r[0, 0]))
    return np.array([rx, ry, rz])


# ---------------------------------------------------------------------------
# rigid transforms as (q, t)


def rigid(q=None, t=None):
    q = np.array([1.0, 0.0, 0.0, 0.0]) if q is None else np.asarray(q, dtype=_F64)
    t = np.zeros(3) if t is None else np.asarray(t, dtype=_F64)
    return q, t


def compose(a, b):
    """a after b."""
    qa, ta = a
    qb, tb = b
    return qnormalize(qmul(qa, qb)), qrotate(qa, tb) + ta


def invert(a):
    q, t = a
    qi = qconj(q)
    return qi, -qrotate(qi, t)


def matrix4(a) -> np.ndarray:
    q, t = a
    m = np.eye(4)
    m[:3, :3] = qmatrix(q)
    m[:3, 3] = t
    return m


# ---------------------------------------------------------------------------
# skeleton / pose / FK


def wrap_angles(a) -> np.ndarray:
    """Radians into (-pi, pi], same arithmetic as the reference Pose."""
    return np.pi - np.mod(np.pi - np.asarray(a, dtype=_F64), 2.0 * np.pi)


@dataclass(frozen=True)
class PoseSpec:
    """Mirror of the reference Pose (rigging.py:70-104): joint Euler angles
    are wrapped once at construction, exactly like Pose.__post_init__."""

    joint_rotations: np.ndarray
    global_rotation: np.ndarray
    global_translation: np.ndarray

    @staticmethod
    def make(euler, g_rot=None, g_trans=None) -> "PoseSpec":
        r = np.asarray(euler, dtype=_F64)
        q = np.array([1.0, 0.0, 0.0, 0.0]) if g_rot is None else np.asarray(g_rot, dtype=_F64)
        t = np.zeros(3) if g_trans is None else np.asarray(g_trans, dtype=_F64)
        if r.ndim != 2 or r.shape[1] != 3:
            raise ContractViolation("joint_rotations must be (J, 3)")
        if not (np.isfinite(r).all() and np.isfinite(q).all() and np.isfinite(t).all()):
            raise ContractViolation("pose contains non-finite values")
        return PoseSpec(wrap_angles(r), q, t)

    @staticmethod
    def from_any(pose) -> "PoseSpec":
        """A reference Pose (already wrapped) or a PoseSpec passes through."""
        if isinstance(pose, PoseSpec):
            return pose
        return PoseSpec(np.asarray(pose.joint_rotations, dtype=_F64),
                        np.asarray(pose.global_rotation, dtype=_F64),
                        np.asarray(pose.global_translation, dtype=_F64))


@dataclass(frozen=True)
class Rig:
    """Parents-first joint tree with bind-pose locals (translation-only or
    full rigid), the data the reference ``Skeleton`` carries."""

    parents: np.ndarray            # (J,) int32, -1 for the root
    bind_q: np.ndarray             # (J, 4)
    bind_t: np.ndarray             # (J, 3)

    @property
    def n_joints(self) -> int:
        return int(self.parents.shape[0])

    @staticmethod
    def from_any(skel) -> "Rig":
        """Accept a Rig or an object shaped like animvox.rigging.Skeleton."""
        if isinstance(skel, Rig):
            return skel
        return Rig(parents=np.asarray(skel.parents, dtype=np.int32),
                   bind_q=np.stack([np.asarray(b.rotation, dtype=_F64) for b in skel.bind_local]),
                   bind_t=np.stack([np.asarray(b.translation, dtype=_F64) for b in skel.bind_local]))

    def bind_locals(self):
        return [(np.asarray(self.bind_q[j], dtype=_F64), np.asarray(self.bind_t[j], dtype=_F64))
                for j in range(self.n_joints)]


def forward_kinematics(rig: Rig, pose: PoseSpec):
    """Global joint transforms (list of (q, t)) for a wrapped pose."""
    euler = np.asarray(pose.joint_rotations, dtype=_F64)
    if euler.shape != (rig.n_joints, 3):
        raise ContractViolation(f"pose has {euler.shape[0]} joints, skeleton has {rig.n_joints}")
    g = rigid(pose.global_rotation, pose.global_translation)
    zero = np.zeros(3)
    locals_ = rig.bind_locals()
    out = []
    for j in range(rig.n_joints):
        local = compose(locals_[j], (q_from_euler_xyz(euler[j]), zero))
        p = int(rig.parents[j])
        out.append(compose(g if p == -1 else out[p], local))
    return out


def canonical_globals(rig: Rig):
    return forward_kinematics(rig, PoseSpec.make(np.zeros((rig.n_joints, 3))))


@dataclass(frozen=True)
class PoseTables:
    """Per-joint tables a frame needs on the device (rigging.py:343-347)."""

    delta_mats: np.ndarray   # (J, 4, 4) posed * canonical^-1
    delta_quats: np.ndarray  # (J, 4)
    rot_inv: np.ndarray      # (J, 3, 3) R(conj(delta q))

    @property
    def affine34(self) -> np.ndarray:
        """(J, 12) row-major 3x4 blocks, the warp kernel's joint table."""
        return np.ascontiguousarray(self.delta_mats[:, :3, :].reshape(-1, 12))


def pose_tables(rig: Rig, pose: PoseSpec, canonical=None) -> PoseTables:
    posed = forward_kinematics(rig, pose)
    canon = canonical if canonical is not None else canonical_globals(rig)
    deltas = [compose(p, invert(c)) for p, c in zip(posed, canon)]
    return PoseTables(
        delta_mats=np.stack([matrix4(d) for d in deltas]),
        delta_quats=np.stack([d[0] for d in deltas]),
        rot_inv=np.stack([qmatrix(qconj(d[0])) for d in deltas]),
    )


class NativePoseTables:
    """pose_tables() through the native restatement (artemis_host_pose_tables,
    csrc/hostfk.cu): the same doubles in microseconds instead of ~1.4 ms of
    tiny numpy calls per 24-joint pose. Used only where agrees() holds -- a
    once-per-process bit-for-bit comparison with the numpy restatement above
    on seeded random rigs and poses (the two BLAS reductions numpy dispatches
    to are the part that could differ between hosts)."""

    _agree: bool | None = None

    def __init__(self, rig: Rig, canonical=None):
        self.rig = rig
        canon = canonical if canonical is not None else canonical_globals(rig)
        self.parents = np.ascontiguousarray(rig.parents, dtype=np.int32)
        self.bind_q = np.ascontiguousarray(rig.bind_q, dtype=_F64)
        self.bind_t = np.ascontiguousarray(rig.bind_t, dtype=_F64)
        self.canon_q = np.ascontiguousarray(np.stack([c[0] for c in canon]), dtype=_F64)
        self.canon_t = np.ascontiguousarray(np.stack([c[1] for c in canon]), dtype=_F64)

    def __call__(self, pose: PoseSpec) -> PoseTables:
        from . import _lib

        J = self.rig.n_joints
        euler = np.ascontiguousarray(pose.joint_rotations, dtype=_F64)
        if euler.shape != (J, 3):
            raise ContractViolation(f"pose has {euler.shape[0]} joints, skeleton has {J}")
        gq = np.ascontiguousarray(pose.global_rotation, dtype=_F64)
        gt = np.ascontiguousarray(pose.global_translation, dtype=_F64)
        dm = np.empty((J, 4, 4))
        dq = np.empty((J, 4))
        ri = np.empty((J, 3, 3))
        P = lambda a: a.ctypes.data  # noqa: E731
        rc = _lib.load_library().artemis_host_pose_tables(J, P(self.parents), P(self.bind_q),
                                                   P(self.bind_t), P(euler), P(gq), P(gt),
                                                   P(self.canon_q), P(self.canon_t), P(dm), P(dq),
                                                   P(ri))
        if rc != 0:
            raise ContractViolation("zero quaternion or invalid rig in forward kinematics")
        return PoseTables(delta_mats=dm, delta_quats=dq, rot_inv=ri)

    @classmethod
    def agrees(cls) -> bool:
        if cls._agree is None:
            rng = np.random.default_rng(20220211)
            ok = True
            for trial in range(8):
                J = 24
                parents = np.array([-1] + [int(rng.integers(0, j)) for j in range(1, J)], np.int32)
                bq = rng.standard_normal((J, 4))
                bq /= np.linalg.norm(bq, axis=1, keepdims=True)
                rig = Rig(parents=parents, bind_q=bq, bind_t=rng.standard_normal((J, 3)) * 0.3)
                canon = canonical_globals(rig)
                native = cls(rig, canon)
                for _ in range(4):
                    g = rng.standard_normal(4)
                    pose = PoseSpec.make(rng.uniform(-4, 4, (J, 3)), g / np.linalg.norm(g),
                                         rng.standard_normal(3))
                    a = pose_tables(rig, pose, canonical=canon)
                    b = native(pose)
                    ok &= all(x.tobytes() == y.tobytes() for x, y in
                              ((a.delta_mats, b.delta_mats), (a.delta_quats, b.delta_quats),
                               (a.rot_inv, b.rot_inv)))
            cls._agree = bool(ok)
        return cls._agree


def identity_tables() -> PoseTables:
    """The no-warp case (identity_warp, rigging.py:400-416)."""
    return PoseTables(
        delta_mats=np.eye(4)[None].copy(),
        delta_quats=np.array([[1.0, 0.0, 0.0, 0.0]]),
        rot_inv=np.eye(3)[None].copy(),
    )


# ---------------------------------------------------------------------------
# cameras


@dataclass(frozen=True)
class PinholeCamera:
    """Pinhole intrinsics plus the world-to-camera rigid transform."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    w2c_q: np.ndarray
    w2c_t: np.ndarray

    def cam_to_world(self):
        """(R (3,3), origin (3,)) as rays_for_camera derives them."""
        q, t = invert((self.w2c_q, self.w2c_t))
        return qmatrix(q), t

    def scaled(self, width: int, height: int) -> "PinholeCamera":
        """render._scaled_camera (render.py:129-143)."""
        sx = width / self.width
        sy = height / self.height
        return PinholeCamera(self.fx * sx, self.fy * sy, self.cx * sx, self.cy * sy,
                             width, height, self.w2c_q, self.w2c_t)

    @staticmethod
    def from_any(cam) -> "PinholeCamera":
        """Accept a PinholeCamera or any object shaped like animvox.Camera."""
        if isinstance(cam, PinholeCamera):
            return cam
        w2c = cam.world_to_camera
        return PinholeCamera(float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
                             int(cam.width), int(cam.height),
                             np.asarray(w2c.rotation, dtype=_F64),
                             np.asarray(w2c.translation, dtype=_F64))


def look_at(position, target, width: int, height: int, focal: float,
            up=(0.0, 0.0, 1.0)) -> PinholeCamera:
    position = np.asarray(position, dtype=_F64)
    fwd = np.asarray(target, dtype=_F64) - position
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=_F64))
    norm = np.linalg.norm(right)
    if norm < 1e-9:
        raise ContractViolation("view direction is parallel to the up axis")
    right /= norm
    down = np.cross(fwd, right)
    c2w = np.eye(4)
    c2w[:3, :3] = np.stack([right, down, fwd], axis=1)
    c2w[:3, 3] = position
    q, t = invert((q_from_matrix(c2w[:3, :3]), c2w[:3, 3].copy()))
    return PinholeCamera(focal, focal, width / 2.0, height / 2.0, width, height, q, t)


def orbit(azimuth: float, elevation: float, radius: float, width: int, height: int,
          focal: float, target=(0.0, 0.0, 0.0)) -> PinholeCamera:
    if radius <= 0:
        raise ContractViolation("orbit radius must be positive")
    target = np.asarray(target, dtype=_F64)
    pos = target + radius * np.array(
        [np.cos(elevation) * np.cos(azimuth), np.cos(elevation) * np.sin(azimuth),
         np.sin(elevation)]
    )
    return look_at(pos, target, width, height, focal)


def focal_for_fov(width: int, fov_deg: float) -> float:
    """D7: the configs state a horizontal fov, the reference a focal."""
    return (width / 2.0) / math.tan(math.radians(fov_deg) / 2.0)
