"""Edge cases of the device frame pipeline against the CPU oracle (which is
pinned to the reference by tests/test_oracle_golden.py): image sizes that
are not whole 8x4 tiles, a single pixel, a camera inside the body's box,
rays running exactly along grid planes (zero direction components, origins
on a plane), a one-voxel character, and the exact tree arrays the rebuild
leaves behind in each case. Same bars as the other parity tests: tree and
depth exact, F within 1e-4 max / 1e-5 mean-abs, alpha within 1e-6 (fp32
maps) or 1e-9 (fp64 maps, ARTEMIS_FRAME_MAPS64)."""

from __future__ import annotations

import dataclasses
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2202_05628_b200 import kinematics as KM
from paper_2202_05628_b200 import synthetic as S

pytestmark = pytest.mark.gpu

F_MAX, F_MEAN = 1e-4, 1e-5


@pytest.fixture(scope="module")
def mini():
    return S.make_scene("c0", resolution=64, image=(64, 64))


def frame_vs_oracle(sc, pose, cam, maps64=False, graph=False):
    from paper_2202_05628_b200.frame import FramePipeline

    fp = FramePipeline.from_scene(sc)
    try:
        F, A, D = fp.run(pose, cam, graph=graph, parity=True, maps64=maps64,
                         lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep)
        fp.stream.synchronize()
        if pose is not None:
            want = oracle.render_frame(sc, KM.pose_tables(sc.rig, pose), cam)
        else:  # canonical cells, rotation joint 0, identity inverse rotation
            tree = oracle.build_octree(sc.cells)
            R, origin = cam.cam_to_world()
            og, dg, dw = oracle.camera_rays(R, origin, cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                                            cam.height, sc.lo, sc.cell_size)
            Fw, Aw, Dw = oracle.render_rays(*tree, og, dg, dw, 0.0, np.inf, sc.flut64(),
                                            np.zeros(sc.n_voxels, np.int32),
                                            KM.identity_tables().rot_inv, sc.degree, sc.channels,
                                            sc.lambda_th, sc.sigma_dep, True)
            want = dict(tree=tree, F=Fw, A=Aw, D=Dw)
        codes, fidx, root, left, right, bmin, bsize = want["tree"]
        t = fp.tree()
        assert t["n_live"] == codes.size
        assert np.array_equal(t["codes"], codes) and np.array_equal(t["flut_idx"], fidx)
        assert t["root"] == root
        for k, v in (("left", left), ("right", right), ("box_min", bmin), ("box_size", bsize)):
            assert np.array_equal(t[k], v), k
        Fh = F.cpu().numpy().astype(np.float64)
        err = np.abs(Fh - want["F"])
        assert err.max(initial=0.0) <= F_MAX and err.mean() <= F_MEAN
        Ah, Dh = A.cpu().numpy(), D.cpu().numpy()
        if maps64:
            assert np.max(np.abs(Ah - want["A"]), initial=0.0) <= 1e-9
            assert np.array_equal(Dh, want["D"])
        else:
            assert np.max(np.abs(Ah - want["A"]), initial=0.0) <= 1e-6
            assert np.array_equal(Dh, want["D"].astype(np.float32))
        return want
    finally:
        fp.close()


@pytest.mark.parametrize("size", [(37, 23), (1, 1), (9, 5), (8, 4)])
def test_image_not_whole_tiles(mini, size):
    W, H = size
    cam = KM.orbit(math.radians(30.0), math.radians(10.0), 2.5, W, H,
                   KM.focal_for_fov(max(W, 8), 40.0))
    frame_vs_oracle(mini, KM.PoseSpec.make(mini.poses[0]), cam)


@pytest.mark.parametrize("maps64", [False, True])
def test_camera_inside_the_body_box(mini, maps64):
    """Rays start inside the leaf AABB (the walk's first cell comes from the
    origin, not from an AABB entry)."""
    cam = KM.look_at([0.05, -0.03, 0.02], [1.0, 0.3, 0.1], 48, 40, KM.focal_for_fov(48, 90.0))
    want = frame_vs_oracle(mini, KM.PoseSpec.make(mini.poses[0]), cam, maps64=maps64)
    assert (want["A"] > 0).any()


def test_rays_along_grid_planes(mini):
    """Camera on the x axis looking down -x with an odd image: the centre
    column/row rays have exactly zero y/z direction components and grid
    origins exactly on cell planes (og = 32), the slab test's d == 0
    branch; every other ray crosses planes at exactly tied distances
    along the image diagonals."""
    cam = KM.look_at([2.5, 0.0, 0.0], [0.0, 0.0, 0.0], 33, 33, KM.focal_for_fov(33, 40.0))
    R, origin = cam.cam_to_world()
    og, dg, dw = oracle.camera_rays(R, origin, cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                                    cam.height, mini.lo, mini.cell_size)
    assert (dg[:, 1] == 0.0).any() and (dg[:, 2] == 0.0).any()
    assert og[0, 1] == np.floor(og[0, 1])
    want = frame_vs_oracle(mini, None, cam)
    assert (want["A"] > 0).any()


def test_axis_aligned_camera_posed(mini):
    cam = KM.look_at([0.0, -2.5, 0.0], [0.0, 0.0, 0.0], 33, 31, KM.focal_for_fov(33, 40.0))
    frame_vs_oracle(mini, KM.PoseSpec.make(mini.poses[0]), cam, graph=True)


def test_single_voxel_character(mini):
    """One voxel: the tree is the lone leaf (root = ~0, no internal nodes)."""
    i = mini.n_voxels // 2
    sc = dataclasses.replace(mini, cells=mini.cells[i:i + 1].copy(),
                             flut32=mini.flut32[i:i + 1].copy(),
                             skin_idx=mini.skin_idx[i:i + 1].copy(),
                             skin_w=mini.skin_w[i:i + 1].copy())
    c = sc.centers()[0]
    cam = KM.look_at(c + np.array([0.0, -1.0, 0.0]), c, 17, 17, KM.focal_for_fov(17, 5.0))
    want = frame_vs_oracle(sc, None, cam)
    assert want["tree"][2] == ~0
    assert (want["A"] > 0).any()


def test_tile_order_does_not_change_the_maps(mini):
    """The render order of the ray tiles (calibrated row-major / centre-out,
    or any permutation) changes only the speed: maps are bit-identical."""
    from paper_2202_05628_b200.frame import FramePipeline

    fp = FramePipeline.from_scene(mini)
    try:
        pose = KM.PoseSpec.make(mini.poses[0])
        cam = KM.orbit(math.radians(20.0), math.radians(15.0), 2.5, 61, 45, KM.focal_for_fov(61, 40.0))
        ref = [x.clone() for x in fp.run(pose, cam, graph=False)]
        n = ((61 + 7) // 8) * ((45 + 3) // 4)
        for seed in (0, 1):
            fp.set_tile_order(61, 45, np.random.default_rng(seed).permutation(n))
            for graph in (False, True):
                got = fp.run(pose, cam, graph=graph)
                fp.stream.synchronize()
                assert all(torch.equal(a, b) for a, b in zip(ref, got))
        with pytest.raises(Exception):
            fp.set_tile_order(61, 45, np.zeros(n, np.int32))  # not a permutation
    finally:
        fp.close()


@pytest.mark.parametrize("maps64", [False, True])
def test_views_in_one_launch_equal_separate_renders(maps64):
    """run_views (one render launch, the views' tiles interleaved) gives
    each view exactly what its own render gives."""
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c1", resolution=64, image=(53, 37))
    fp = FramePipeline.from_scene(sc)
    try:
        pose = KM.PoseSpec.make(sc.poses[0])
        cams = sc.cameras[0][:5]
        sep = []
        for i, cam in enumerate(cams):
            sep.append([x.clone() for x in fp.run(pose, cam, graph=False, maps64=maps64,
                                                   reuse_tree=i > 0)])
        for graph in (False, True, True):
            got = fp.run_views(pose, cams, graph=graph, maps64=maps64)
            fp.stream.synchronize()
            for a, b in zip(sep, got):
                assert all(torch.equal(x, y) for x, y in zip(a, b))
    finally:
        fp.close()


def test_configs1_views_one_launch_full_size():
    """configs[1] at full size: the 8 views rendered in one launch equal
    their separate renders bit for bit."""
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c1")
    fp = FramePipeline.from_scene(sc)
    try:
        pose = KM.PoseSpec.make(sc.poses[0])
        sep = [[x.clone() for x in fp.run(pose, cam, graph=False, reuse_tree=i > 0)]
               for i, cam in enumerate(sc.cameras[0])]
        got = fp.run_views(pose, sc.cameras[0], graph=True)
        fp.stream.synchronize()
        assert len(got) == 8
        for a, b in zip(sep, got):
            assert all(torch.equal(x, y) for x, y in zip(a, b))
    finally:
        fp.close()


@pytest.mark.parametrize("nan_rows", [False, True])
def test_counting_rebuild_equals_sort_path(monkeypatch, nan_rows):
    """The frame pipeline's counting rebuild (rebuild.cu: dense brick masks,
    commutative integer atomics) and its onesweep sort + resolve path
    (ARTEMIS_COUNTING=0) give the same tree, winners, brick walk and maps,
    also with NaN densities (np.lexsort's NaN-last order) -- and both equal
    the oracle's rebuild."""
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c3", resolution=128, shell=3, scale=0.76, channels=16,
                      image=(160, 120), frames=3)
    if nan_rows:
        fl = sc.flut32.copy()
        fl[::97, -1] = np.nan
        sc.flut32 = fl
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ARTEMIS_COUNTING", mode)
        fp = FramePipeline.from_scene(sc)
        res = []
        for f in range(3):
            pose = KM.PoseSpec.make(sc.poses[f])
            F, A, D = fp.run(pose, sc.cameras[f][0], graph=f > 0, parity=True)
            fp.stream.synchronize()
            res.append((fp.tree(), F.clone(), A.clone(), D.clone()))
        fp.close()
        out[mode] = res
    for f in range(3):
        (t1, F1, A1, D1), (t0, F0, A0, D0) = out["1"][f], out["0"][f]
        for k in ("codes", "flut_idx", "left", "right", "box_min", "box_size",
                  "rotation_joint"):
            assert np.array_equal(t1[k], t0[k]), (f, k)
        assert t1["n_live"] == t0["n_live"] and t1["n_in"] == t0["n_in"]
        for a, b in ((F1, F0), (A1, A0), (D1, D0)):  # bit-identical, NaN where NaN
            assert bool(((a == b) | (torch.isnan(a) & torch.isnan(b))).all())
        tables = KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[f]))
        want = oracle.render_frame(sc, tables, sc.cameras[f][0], render=False,
                                   flut64=sc.flut32[:, -1:].astype(np.float64))
        assert np.array_equal(t1["codes"], want["tree"][0])
        assert np.array_equal(t1["flut_idx"], want["tree"][1])


def test_fast_division_path_equals_ddiv(monkeypatch):
    """Camera frames whose operands are in div_fast's range compute every
    plane crossing and camera-ray division as a reciprocal-corrected
    product (bricks.cuh); ARTEMIS_FAST_DIV=0 forces __ddiv_rn. Same maps,
    bit for bit, for single views, multi-view launches and tile shards; a
    camera outside the range (subnormal principal point) falls back by itself
    and still matches the oracle."""
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c1", frames=1, image=(120, 88))
    pose = KM.PoseSpec.make(sc.poses[0])
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ARTEMIS_FAST_DIV", mode)
        fp = FramePipeline.from_scene(sc)
        res = [x.clone() for x in fp.run(pose, sc.cameras[0][1], graph=False)]
        res += [x.clone() for x in fp.run(pose, sc.cameras[0][2], graph=True)]
        res += [x for v in fp.render_views(pose, sc.cameras[0][:3], graph=False) for x in v]
        res += [x.clone() for x in fp.run(pose, sc.cameras[0][5], graph=False, tiles=(0, 2))]
        fp.stream.synchronize()
        out[mode] = res
        fp.close()
    for a, b in zip(out["1"], out["0"]):
        assert torch.equal(a, b)
    monkeypatch.delenv("ARTEMIS_FAST_DIV")
    cam = dataclasses.replace(sc.cameras[0][0], cx=5e-324)
    fp = FramePipeline.from_scene(sc)
    F, A, D = fp.run(pose, cam, graph=False)
    fp.stream.synchronize()
    tables = KM.pose_tables(sc.rig, pose)
    want = oracle.render_frame(sc, tables, cam)
    err = np.abs(F.cpu().numpy().astype(np.float64) - want["F"])
    assert err.max() <= 1e-4 and err.mean() <= 1e-5
    assert np.array_equal(D.cpu().numpy(), want["D"].astype(np.float32))
    fp.close()


def test_api_fast_division_equals_ddiv(monkeypatch):
    """The flat-array API path (render_rays / forward_fit on the brick walk)
    takes the reciprocal-corrected division when the rays' operand ranges
    qualify (kernels.fast_div_ok); forcing __ddiv_rn gives the same bits."""
    from paper_2202_05628_b200 import kernels as K

    sc = S.make_scene("c0", frames=1, image=(96, 96))
    tables = KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[0]))
    fr = oracle.render_frame(sc, tables, sc.cameras[0][0], render=False)
    args = (*fr["tree"], fr["origins_g"], fr["dirs_g"], fr["dirs_w"], 0.0, np.inf, sc.flut32,
            fr["rotation_joint"], tables.rot_inv, sc.degree, sc.channels)
    assert K.fast_div_ok(fr["origins_g"], fr["dirs_g"])
    fast = (*K.render_rays(*args, sc.lambda_th, sc.sigma_dep, True), *K.forward_fit(*args))
    monkeypatch.setattr(K, "fast_div_ok", lambda og, dg: False)
    slow = (*K.render_rays(*args, sc.lambda_th, sc.sigma_dep, True), *K.forward_fit(*args))
    for a, b in zip(fast, slow):
        assert np.array_equal(a, b)
    assert not K.fast_div_ok(np.array([[1e-320, 1.0, 2.0]]), np.ones((1, 3)))
    assert not K.fast_div_ok(np.ones((1, 3)), np.array([[1e-200, 0.0, 1.0]]))


def _opaque(sc, gain=64.0):
    """The configs' densities (softplus(N(0,1)) over half-voxel steps) leave
    every pixel's alpha below ~0.35, so no ray ever stops early; scaled by
    `gain` the body is opaque within a few hits."""
    fl = sc.flut32.copy()
    fl[:, -1] *= np.float32(gain)
    return dataclasses.replace(sc, flut32=fl)


@pytest.mark.parametrize("lambda_th,sigma_dep", [(0.01, 5.0), (0.3, 1.0), (1e-12, 0.0)])
def test_early_stop_thresholds_against_oracle(mini, lambda_th, sigma_dep):
    """The warp-level early ray termination at other thresholds than the
    configs' 1e-4 (the reference's default 0.01, a coarse 0.3 that stops most
    rays after a few hits, and 1e-12 = never) and depth thresholds (a voxel
    registers in the depth map above sigma_dep, render.py:40-42)."""
    sc = dataclasses.replace(_opaque(mini), lambda_th=lambda_th, sigma_dep=sigma_dep)
    want = frame_vs_oracle(sc, KM.PoseSpec.make(sc.poses[0]), sc.cameras[0][0], maps64=True)
    if lambda_th < 1.0e-6:
        assert (want["A"] > 0.99).any()  # the body is opaque: the other thresholds do stop rays


@pytest.mark.parametrize("config", ["c0", "c2"])
def test_early_stop_alpha_drift_bounded_full_size(config):
    """The reference's acceptance property (test_acceptance.py:183-209) at
    configs[0]'s and configs[2]'s full size: stopping once alpha exceeds 1 - lambda_th moves
    every pixel's alpha down by less than lambda_th, never up; a larger
    threshold never integrates further; depth only loses hits."""
    from paper_2202_05628_b200.frame import FramePipeline

    sc = _opaque(S.make_scene(config))
    fp = FramePipeline.from_scene(sc)
    try:
        pose, cam = KM.PoseSpec.make(sc.poses[0]), sc.cameras[0][0]
        maps = {}
        for lam in (1e-12, 1e-4, 0.01, 0.3):
            F, A, D = fp.run(pose, cam, graph=False, maps64=True, lambda_th=lam,
                             sigma_dep=sc.sigma_dep)
            fp.stream.synchronize()
            maps[lam] = (F.cpu().numpy().copy(), A.cpu().numpy().copy(), D.cpu().numpy().copy())
        A_full = maps[1e-12][1]
        assert A_full.max() <= 1.0 and (A_full > 0.99).any()
        prev = A_full
        for lam in (1e-4, 0.01, 0.3):
            A = maps[lam][1]
            drift = A_full - A
            assert drift.min() >= 0.0 and drift.max() < lam, (lam, drift.min(), drift.max())
            assert np.all(A <= prev)
            stopped = A != A_full
            assert np.all(A[stopped] > 1.0 - lam)
            # a ray that stopped early keeps every depth hit it had reached
            D, D_full = maps[lam][2], maps[1e-12][2]
            assert np.all((D == D_full) | np.isinf(D))
            prev = A
        assert (maps[0.3][1] != A_full).any()
    finally:
        fp.close()
