"""The kernel-contract shim's device cache ("device-
cached tree and FLUT keyed by array identity plus a content check, no
per-call re-upload"). The reference calls kernels.render_rays once per ray
in integrate_ray (render.py:209-231) and forward_fit once per batch in fit
(fit.py:474-480); repeated calls on the same FLUT and tree must not move
the FLUT over PCIe again, and an in-place edit of the FLUT must still take
effect on the next call, as it does in the reference."""

from __future__ import annotations

import time

import numpy as np
import pytest

import oracle
from paper_2202_05628_b200 import kinematics as KM
from paper_2202_05628_b200 import synthetic as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2202_05628_b200 import kernels

    kernels.invalidate_cache()
    yield kernels
    kernels.invalidate_cache()


def posed(sc):
    tables = KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[0]))
    fr = oracle.render_frame(sc, tables, sc.cameras[0][0], render=False,
                             flut64=sc.flut32[:, -1:].astype(np.float64))
    return tables, fr


def hit_rays(fr, n):
    """`n` camera rays that see the character (plus their indices)."""
    cnt = oracle.count_hits(*fr["tree"], fr["origins_g"], fr["dirs_g"], 0.0, np.inf)
    idx = np.flatnonzero(cnt > 0)[:: max(1, int((cnt > 0).sum()) // n)][:n]
    return idx


def test_repeated_calls_reuse_device_copies(K):
    """configs[2] FLUT (984,792 x 289 fp64, 2.28 GB): the first render_rays
    uploads it, the next calls (render_rays, forward_fit, single rays) move
    only their rays."""
    sc = S.make_scene("c2")
    tables, fr = posed(sc)
    flut = sc.flut64()
    rj = fr["rotation_joint"]
    idx = hit_rays(fr, 64)
    og, dg, dw = fr["origins_g"], fr["dirs_g"], fr["dirs_w"]
    common = (0.0, np.inf, flut, rj, tables.rot_inv, sc.degree, sc.channels)
    K.cache_stats(reset=True)
    F0, A0, D0 = K.render_rays(*fr["tree"], og[idx], dg[idx], dw[idx], *common, sc.lambda_th,
                               sc.sigma_dep, True)
    s0 = K.cache_stats()
    assert s0["misses"] == 2 and s0["h2d_bytes"] >= flut.nbytes
    times = []
    for r in idx[:16]:  # integrate_ray-style: one call per ray
        t = time.perf_counter()
        F1, A1, D1 = K.render_rays(*fr["tree"], og[r:r + 1], dg[r:r + 1], dw[r:r + 1], *common,
                                   sc.lambda_th, sc.sigma_dep, True)
        times.append(time.perf_counter() - t)
        j = int(np.flatnonzero(idx == r)[0])
        assert np.array_equal(D1, D0[j:j + 1]) and np.array_equal(A1, A0[j:j + 1])
        assert np.array_equal(F1, F0[j:j + 1])
    s1 = K.cache_stats()
    assert s1["misses"] == s0["misses"] and s1["h2d_bytes"] == s0["h2d_bytes"]
    assert s1["hits"] == s0["hits"] + 2 * 16
    K.forward_fit(*fr["tree"], og[idx], dg[idx], dw[idx], *common)
    K.traverse_ray(*fr["tree"], og[idx[0]], dg[idx[0]], 0.0, np.inf)
    s2 = K.cache_stats()
    # forward_fit reuses both; traverse_ray builds its trace-only table once
    assert s2["h2d_bytes"] - s1["h2d_bytes"] < flut.nbytes // 50
    print(f"\nper-call render_rays (1 ray, configs[2] FLUT 2.28 GB, content-checked): "
          f"median {np.median(times) * 1e3:.1f} ms")


def test_in_place_edit_takes_effect(K):
    """The reference re-reads the FLUT on every call: edit densities and
    coefficients in place between two calls -> the second call must see it."""
    sc = S.make_scene("c0")
    tables, fr = posed(sc)
    flut = sc.flut64()
    rj = fr["rotation_joint"]
    idx = hit_rays(fr, 200)
    rays = (fr["origins_g"][idx], fr["dirs_g"][idx], fr["dirs_w"][idx])
    args = lambda: (*fr["tree"], *rays, 0.0, np.inf, flut, rj, tables.rot_inv, sc.degree,  # noqa
                    sc.channels, sc.lambda_th, sc.sigma_dep, True)
    F0, A0, _ = K.render_rays(*args())
    _, _, off, hidx, _, _ = K.forward_fit(*args()[:17])
    leaf = int(hidx[0])
    flut[leaf, -1] *= 7.0  # like FLUT.clamp_densities / SparseAdam.step: in place
    flut[leaf, 0] += 0.25
    F1, A1, D1 = K.render_rays(*args())
    Fw, Aw, Dw = oracle.render_rays(*args())
    assert not np.array_equal(A1, A0)
    assert np.max(np.abs(A1 - Aw)) <= 1e-9 and np.array_equal(D1, Dw)
    assert np.max(np.abs(F1 - Fw)) <= 1e-4
    # identity policy: same buffer -> stale until invalidated, by contract
    K.set_cache_policy("identity")
    try:
        Fi, Ai, _ = K.render_rays(*args())
        flut[leaf, -1] *= 3.0
        Fs, As, _ = K.render_rays(*args())
        assert np.array_equal(As, Ai)  # documented: caller must invalidate
        K.invalidate_cache()
        Fn, An, _ = K.render_rays(*args())
        assert not np.array_equal(An, Ai)
    finally:
        K.set_cache_policy("content")


def test_device_assets_see_in_place_flut_edit(K):
    """render_frame's resident pipelines (pipeline.DEVICE_ASSETS) are keyed
    by the same full-content digest."""
    from paper_2202_05628_b200 import pipeline as P

    sc = S.make_scene("c0", resolution=64, image=(64, 64))

    class Vox:
        cells = sc.cells
        resolution = sc.resolution

        class bounds:
            lo = sc.lo
            hi = sc.hi

    fl = sc.flut64()
    a = P.DEVICE_ASSETS
    a.clear()

    class Asset:
        voxels = Vox
        skeleton = None
        weights = None

        class flut:
            data = fl
            degree = sc.degree
            channels = sc.channels

    fp1 = a.get(Asset)
    assert a.get(Asset) is fp1
    fl[3, 0] = np.nextafter(fl[3, 0], 1.0)
    fp2 = a.get(Asset)
    assert fp2 is not fp1
    a.clear()
