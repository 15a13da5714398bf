"""Race detection without compute-sanitizer (closed on this GPU pool): the
reference's own race check is determinism -- identical results at every
thread count (_core.pyx:6-9, pkg/tests/test_backend.py:17). Here every map
must be bit-identical whatever the persistent render grid (1 CTA ... the
full machine: different ray-to-warp schedules, different interleavings of
the shared-memory queue protocols and the atomic ray queue) and over
repeated runs; the onesweep sort's decoupled look-back must give the same
permutation on every repeat. scripts/gpu_checks.sh also runs these and the
parity suites on the bounds-checking build (-DARTEMIS_DEBUG_CHECKS)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2202_05628_b200 import _lib
from paper_2202_05628_b200 import kernels as K
from paper_2202_05628_b200 import kinematics as KM
from paper_2202_05628_b200 import synthetic as S

pytestmark = pytest.mark.gpu

CAPS = (1, 3, 37, 0)


@pytest.fixture
def cap():
    L = _lib.lib()

    def set_cap(n):
        assert L.artemis_debug_set_render_blocks(n) == 0

    yield set_cap
    set_cap(0)


def test_camera_mode_schedule_independent(cap):
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c0", frames=2, image=(200, 152))
    fp = FramePipeline.from_scene(sc)
    pose = KM.PoseSpec.make(sc.poses[1])
    cam = sc.cameras[1][0]
    ref = None
    for c in CAPS:
        cap(c)
        for _ in range(2):
            out = [x.clone() for x in fp.run(pose, cam, graph=False, lambda_th=sc.lambda_th,
                                             sigma_dep=sc.sigma_dep)]
            fp.stream.synchronize()
            if ref is None:
                ref = out
            for a, b in zip(out, ref):
                assert torch.equal(a, b), c
    assert (ref[1] > 0).sum() > 1000
    fp.close()


@pytest.mark.parametrize("mode", ["walk", "dfs"])
def test_api_mode_schedule_independent(cap, mode):
    sc = S.make_scene("c0", frames=1, image=(128, 128))
    tables = KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[0]))
    fr = oracle.render_frame(sc, tables, sc.cameras[0][0], render=False)
    old = K.DeviceTree.MAX_BRICK_TABLE
    K.DeviceTree.MAX_BRICK_TABLE = 0 if mode == "dfs" else old
    try:
        args = (*fr["tree"], fr["origins_g"], fr["dirs_g"], fr["dirs_w"], 0.0, np.inf,
                sc.flut32, fr["rotation_joint"], tables.rot_inv, sc.degree, sc.channels)
        ref = None
        for c in CAPS:
            cap(c)
            out = (*K.render_rays(*args, sc.lambda_th, sc.sigma_dep, True),
                   *K.forward_fit(*args))
            if ref is None:
                ref = out
            for a, b in zip(out, ref):
                assert np.array_equal(a, b), c
    finally:
        K.DeviceTree.MAX_BRICK_TABLE = old
        K.invalidate_cache()


def test_multiview_and_sharded_schedule_independent(cap):
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c1", frames=1, image=(96, 80))
    fp = FramePipeline.from_scene(sc)
    pose = KM.PoseSpec.make(sc.poses[0])
    ref = None
    for c in CAPS:
        cap(c)
        views = fp.render_views(pose, sc.cameras[0][:4], graph=False)
        shard = [x.clone() for x in fp.run(pose, sc.cameras[0][2], graph=False, tiles=(1, 3))]
        fp.stream.synchronize()
        out = [x for v in views for x in v] + shard
        if ref is None:
            ref = out
        for a, b in zip(out, ref):
            assert torch.equal(a, b), c
    fp.close()


@pytest.mark.parametrize("bits", [30, 63])
def test_sort_lookback_repeatable(bits):
    rng = np.random.default_rng(bits)
    keys = rng.integers(0, 1 << bits, size=1_500_017, dtype=np.int64).astype(np.uint64)
    keys[::7] = keys[0]  # long duplicate runs: stability under the look-back
    want = oracle.sort_order(keys)
    for _ in range(5):
        assert np.array_equal(K.sort_order(keys), want)


def test_reciprocal_corrected_division_is_exact():
    """The cell walk computes every plane crossing fl((k - o) / d) as
    RN(q + (n - q d) r), q = RN(n r), r = RN(1/d) (bricks.cuh crossing);
    Markstein's theorem makes that __ddiv_rn's result. 2^28 samples over
    walk-like, adversarial-significand, near-multiple and wide random
    operands must agree bit for bit (the config-scale trace digests in
    test_gpu_traces.py pin it on the real walk)."""
    import ctypes

    L = _lib.lib()
    bad = ctypes.c_ulonglong(0)
    assert L.artemis_debug_division_selftest(1 << 28, 12345, ctypes.byref(bad), None) == 0
    assert bad.value == 0


def test_row_group_ranking_is_exact():
    """Phase C balances its passes by ranking row groups by member count
    (with the L2 row prefetch) when the FLUT is not L2-resident, and by
    splitting groups into items of <= 2 members when it is -- at test sizes
    the automatic decision is "resident". Forcing each decision must give
    bit-identical maps in camera mode, multi-view and API mode (walk + DFS):
    both only regroup the shading of different rays within a level."""
    from paper_2202_05628_b200.frame import FramePipeline

    L = _lib.lib()
    sc = S.make_scene("c1", frames=1, image=(160, 128))
    fp = FramePipeline.from_scene(sc)
    pose = KM.PoseSpec.make(sc.poses[0])
    tables = KM.pose_tables(sc.rig, pose)
    fr = oracle.render_frame(sc, tables, sc.cameras[0][0], render=False)
    old = K.DeviceTree.MAX_BRICK_TABLE
    outs = {}
    try:
        for mode in (1, 0, -1):
            assert L.artemis_debug_set_flut_l2_resident(mode) == 0
            cam = [x.clone() for x in fp.run(pose, sc.cameras[0][1], graph=False,
                                             lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep)]
            views = fp.render_views(pose, sc.cameras[0][:3], graph=False)
            fp.stream.synchronize()
            got = [x.cpu().numpy() for x in cam] + [x.cpu().numpy() for v in views for x in v]
            for enum in ("walk", "dfs"):
                K.DeviceTree.MAX_BRICK_TABLE = 0 if enum == "dfs" else old
                K.invalidate_cache()
                args = (*fr["tree"], fr["origins_g"], fr["dirs_g"], fr["dirs_w"], 0.0, np.inf,
                        sc.flut32, fr["rotation_joint"], tables.rot_inv, sc.degree, sc.channels)
                got += list(K.render_rays(*args, sc.lambda_th, sc.sigma_dep, True))
            outs[mode] = got
    finally:
        assert L.artemis_debug_set_flut_l2_resident(-1) == 0
        K.DeviceTree.MAX_BRICK_TABLE = old
        K.invalidate_cache()
        fp.close()
    assert (outs[1][1] > 0).sum() > 1000
    for mode in (0, -1):
        for a, b in zip(outs[mode], outs[1]):
            assert np.array_equal(a, b), mode
