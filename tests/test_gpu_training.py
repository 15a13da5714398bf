"""GPU training iteration: the device SparseAdam, pair
(VRT) term and L1 gradients against the reference's own output
(tests/golden/fit.npz) bit for bit, and DeviceTrainer.step against a host
loop built from the same GPU forward/backward plus the oracle's restatement
of fit.py's optimiser, bit for bit over several iterations."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2202_05628_b200 import _lib
from paper_2202_05628_b200 import kernels as K
from paper_2202_05628_b200 import kinematics as KM
from paper_2202_05628_b200 import synthetic as S
from paper_2202_05628_b200.device import ptr
from paper_2202_05628_b200.training import DeviceTrainer

pytestmark = pytest.mark.gpu


def dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()


def test_sparse_adam_matches_reference(golden_fit):
    g = golden_fit
    L = _lib.lib()
    p = dev(g["params0"], np.float64)
    m = torch.zeros_like(p)
    v = torch.zeros_like(p)
    n, w = p.shape
    for k in range(3):
        grad = dev(g["grads"][k], np.float64)
        t = dev(g["touches"][k], np.uint8)
        assert L.artemis_sparse_adam(ptr(p), ptr(m), ptr(v), ptr(grad), ptr(t), n, w, 0.05, 0.9,
                                     0.999, 1e-8, 1.0 - 0.9 ** (k + 1), 1.0 - 0.999 ** (k + 1),
                                     None) == 0
    torch.cuda.synchronize()
    assert np.array_equal(p.cpu().numpy(), g["params3"])
    assert np.array_equal(m.cpu().numpy(), g["m3"]) and np.array_equal(v.cpu().numpy(), g["v3"])


def test_density_clamp_covers_untouched_rows():
    """FLUT.clamp_densities (volume.py:166-167) clamps the whole density
    column every iteration: a user-supplied init with negative densities in
    rows no ray touches is clamped too (np.maximum: NaN stays NaN)."""
    L = _lib.lib()
    rng = np.random.default_rng(4)
    n, w = 500, 10
    p0 = rng.normal(size=(n, w))
    p0[7, -1] = np.nan
    touched = (rng.random(n) < 0.3).astype(np.uint8)
    grad = rng.normal(size=(n, w)) * touched[:, None]
    p = dev(p0, np.float64)
    m, v = torch.zeros_like(p), torch.zeros_like(p)
    assert L.artemis_sparse_adam(ptr(p), ptr(m), ptr(v), ptr(dev(grad, np.float64)),
                                 ptr(dev(touched, np.uint8)), n, w, 0.05, 0.9, 0.999, 1e-8,
                                 0.1, 0.001, None) == 0
    got = p.cpu().numpy()
    untouched = touched == 0
    assert np.array_equal(got[untouched, :-1], p0[untouched, :-1])
    want = np.maximum(p0[untouched, -1], 0.0)
    assert np.array_equal(got[untouched, -1], want, equal_nan=True)
    assert np.isnan(got[7, -1]) and (got[:, -1][~np.isnan(got[:, -1])] >= 0).all()


def test_pair_term_matches_np_add_at(golden_fit):
    g = golden_fit
    L = _lib.lib()
    data = dev(g["params0"], np.float64)
    n, w = data.shape
    pairs = dev(g["pairs"], np.int64)
    P = pairs.shape[0]
    grad = torch.zeros_like(data)
    touched = torch.zeros(n, dtype=torch.uint8, device="cuda")
    ws = torch.empty(L.artemis_vrt_workspace_bytes(P, n), dtype=torch.uint8, device="cuda")
    assert L.artemis_vrt_grads(ptr(data), n, w, ptr(pairs), P, 0.01 / (P * w), ptr(grad),
                               ptr(touched), ptr(ws), ws.numel(), None) == 0
    torch.cuda.synchronize()
    assert np.array_equal(grad.cpu().numpy(), g["vrt_grad"])
    assert np.array_equal(touched.cpu().numpy().astype(bool), g["vrt_touched"])


def test_l1_gradients_match_reference(golden_fit):
    g = golden_fit
    L = _lib.lib()
    n, C = g["F"].shape
    F = dev(g["F"], np.float32)
    A = dev(g["A"], np.float64)
    dldf = torch.empty((n, C), dtype=torch.float64, device="cuda")
    dlda = torch.empty(n, dtype=torch.float64, device="cuda")
    lr = torch.empty(n, dtype=torch.float64, device="cuda")
    ls = torch.empty(1, dtype=torch.float64, device="cuda")
    assert L.artemis_l1_grads(ptr(F), ptr(A), ptr(dev(g["gt_f"], np.float64)),
                              ptr(dev(g["gt_a"], np.float64)), n, C, ptr(dldf), ptr(dlda),
                              ptr(lr), ptr(ls), None) == 0
    torch.cuda.synchronize()
    assert np.array_equal(dldf.cpu().numpy(), g["dldf"])
    assert np.array_equal(dlda.cpu().numpy(), g["dlda"])
    assert abs(float(ls.item()) / n - float(g["loss"])) <= 1e-12 * float(g["loss"])


def test_trainer_equals_host_loop():
    sc = S.make_scene("c0", resolution=64, image=(64, 64), channels=3, frames=2)
    tables = KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[0]))
    fr = oracle.render_frame(sc, tables, sc.cameras[0][0], render=False)
    tree, rj, pairs = fr["tree"], fr["rotation_joint"], fr["pairs"]
    og, dg, dw = fr["origins_g"], fr["dirs_g"], fr["dirs_w"]
    rng = np.random.default_rng(9)
    start = sc.flut64().copy()
    target = start.copy()
    target[:, :-1] += rng.normal(scale=0.2, size=target[:, :-1].shape)
    gtF, gtA, *_ = oracle.forward_fit(*tree, og, dg, dw, 0.0, np.inf, target, rj, tables.rot_inv,
                                      sc.degree, sc.channels)
    trainer = DeviceTrainer(start, sc.degree, sc.channels, lambda_vrt=0.01)
    host = start.copy()
    opt = oracle.SparseAdam(host.shape, lr=0.05)
    for it in range(4):
        pick = rng.integers(0, og.shape[0], size=2048)
        args = (og[pick], dg[pick], dw[pick])
        l_rgba, l_vrt = trainer.step(tree, *args, gtF[pick], gtA[pick], rj, tables.rot_inv,
                                     pairs=pairs)
        # host loop: same GPU forward / backward, the reference's bookkeeping
        f, a, off, hi, h0, h1 = K.forward_fit(*tree, *args, 0.0, np.inf, host, rj,
                                              tables.rot_inv, sc.degree, sc.channels)
        dldf, dlda = oracle.l1_grads(f.astype(np.float32), a, gtF[pick], gtA[pick])
        grad = K.backward_rays(off, hi, h0, h1, args[2], rj, tables.rot_inv, host, dldf, dlda,
                               sc.degree, sc.channels)
        touched = np.zeros(host.shape[0], bool)
        touched[np.unique(hi)] = True
        oracle.vrt_add(grad, touched, host, pairs, 0.01)
        opt.step(host, grad, touched)
        assert np.array_equal(trainer.data, host), it
        want = np.mean(np.sum(np.abs(f.astype(np.float32).astype(np.float64) - gtF[pick]), 1)
                       + np.abs(a - gtA[pick]))  # loss_rgba, fit.py:52-68
        assert abs(l_rgba - want) <= 1e-12 * want
        assert l_vrt > 0.0
