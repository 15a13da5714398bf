"""Finite-difference gradient check of the GPU training gradients, the
reference's own probe method (tests/gradcheck.py:74-121 there): on tiny
random volumes (2^3 or 4^3 grids, 3-9 cells, SH degree 0-2, 1 or 3
channels, 8 rays, random per-entry rotations) differentiate a fixed random
linear functional J = sum(w_f F) + sum(w_a alpha) of the traced batch and
compare the analytic backward_rays gradient with central differences
(h = 1e-3) on the entries with the largest gradients plus random ones.

* fp64: analytic = the GPU kernel; J from the fp64 forward (the oracle's
  restatement of forward_fit): max relative error <= 1e-6, the reference's
  own bar for its double instantiation (test_fit.py:241-249).
* fp32: analytic = the GPU kernel's float32 instantiation on the
  f32-rounded FLUT, J from the fp64 forward: <= 1e-3, the reference's
  single-precision bar (test_fit.py:251-257).
* consistency of the GPU's own pair: J from the GPU forward_fit (fp32
  shading, so roundoff ~1e-7 |J|) with h = 1e-2 against the fp64 GPU
  gradient: <= 5e-3.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2202_05628_b200 import kernels as K

pytestmark = pytest.mark.gpu


def random_scene(rng):
    res = int(rng.choice([2, 4]))
    n_cells = int(rng.integers(3, min(9, res ** 3) + 1))
    flat = rng.choice(res ** 3, size=n_cells, replace=False)
    cells = np.stack(np.unravel_index(flat, (res, res, res)), axis=1).astype(np.int32)
    degree = int(rng.integers(0, 3))
    channels = int(rng.choice([1, 3]))
    width = (degree + 1) ** 2 * channels + 1
    data = rng.uniform(-0.5, 0.5, size=(n_cells, width))
    data[:, -1] = rng.uniform(0.1, 3.0, size=n_cells)
    tree = oracle.build_octree(cells)
    origins = rng.uniform(-0.5, 0.0, size=(8, 3))
    dirs = rng.uniform(0.2, 0.8, size=(8, 3)) - origins
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    if rng.random() < 0.5:
        q = rng.standard_normal((3, 4))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        w, x, y, z = q.T
        rot = np.empty((3, 3, 3))
        rot[:, 0] = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1)
        rot[:, 1] = np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1)
        rot[:, 2] = np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1)
        rot_inv = np.ascontiguousarray(rot.transpose(0, 2, 1))
        rot_index = rng.integers(0, 3, size=n_cells).astype(np.int32)
    else:
        rot_index = np.zeros(n_cells, np.int32)
        rot_inv = np.eye(3)[None].copy()
    cell = 1.0 / res  # bounds [0, 1)^3
    og = np.ascontiguousarray(origins / cell)
    dg = np.ascontiguousarray(dirs / cell)
    return tree, data, og, dg, dirs, rot_index, rot_inv, degree, channels


def fd_error(rng, dtype, forward, h=1e-3):
    tree, data, og, dg, dw, ri, ro, degree, channels = random_scene(rng)
    base = data.astype(dtype).astype(np.float64)
    w_f = rng.uniform(-1.0, 1.0, size=(og.shape[0], channels))
    w_a = rng.uniform(-1.0, 1.0, size=og.shape[0])

    def fwd(d):
        return forward(*tree, og, dg, dw, 0.0, np.inf, d, ri, ro, degree, channels)

    def objective(d):
        f, a, *_ = fwd(d)
        return float(np.sum(w_f * f) + np.sum(w_a * a))

    _, _, off, hi, h0, h1 = fwd(base)
    grad = K.backward_rays(off, hi, h0, h1, dw, ri, ro, base.astype(dtype), w_f.astype(dtype),
                           w_a.astype(dtype), degree, channels, True, 1)
    assert grad.dtype == dtype
    touched = np.unique(np.asarray(hi, dtype=np.int64))
    if touched.size == 0:
        return 0.0
    width = base.shape[1]
    coords = [(int(i), c) for i in touched for c in range(width)]
    order = np.argsort([-abs(float(grad[i, c])) for i, c in coords])
    keep = [coords[k] for k in order[:5]]
    extra = rng.choice(len(coords), size=min(5, len(coords)), replace=False)
    keep += [coords[int(k)] for k in extra]
    g_fd, g_an = np.zeros(len(keep)), np.zeros(len(keep))
    for k, (i, c) in enumerate(keep):
        bumped = base.copy()
        bumped[i, c] = base[i, c] + h
        up = objective(bumped)
        bumped[i, c] = base[i, c] - h
        down = objective(bumped)
        g_fd[k] = (up - down) / (2 * h)
        g_an[k] = float(grad[i, c])
    scale = max(1e-12, float(np.max(np.abs(g_fd))))
    return float(np.max(np.abs(g_an - g_fd))) / scale


def test_double_precision_gradients():
    rng = np.random.default_rng(66)
    worst = max(fd_error(rng, np.float64, oracle.forward_fit) for _ in range(40))
    assert worst <= 1e-6, worst


def test_single_precision_gradients():
    rng = np.random.default_rng(77)
    worst = max(fd_error(rng, np.float32, oracle.forward_fit) for _ in range(40))
    assert worst <= 1e-3, worst


def test_gpu_forward_backward_consistent():
    rng = np.random.default_rng(88)
    worst = max(fd_error(rng, np.float64, K.forward_fit, h=1e-2) for _ in range(40))
    assert worst <= 5e-3, worst
