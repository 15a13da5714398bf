"""The remaining BASELINE configs end to end on the GPU against the oracle:
configs[1] (one pose, 8 views of 512^2, warp + rebuild once, one render per
view) and configs[4] at full structure (1024^3 grid, ~4M leaves, 32 joints,
two 1440x1600 stereo eyes sharing one rebuild) -- the maximum-size case.

Bit-exact: the rebuilt tree (codes, FLUT rows, child links, boxes) and the
rotation joints; depth on sampled pixels (fp32 of the exact entry
distance). Tolerance: F 1e-4 max / 1e-5 mean-abs, alpha 1e-6 (fp32 maps).
configs[4] runs at its own 32 channels; the oracle (fp64 FLUT) shades it in
eight 4-channel column slices of the same table (shading is per channel:
slice s holds columns h*32 + 4s .. 4s+3 and the density), so its fp64 copy
stays ~1.2 GB at a time."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2202_05628_b200 import kinematics as KM
from paper_2202_05628_b200 import synthetic as S

pytestmark = pytest.mark.gpu

F_MAX, F_MEAN = 1e-4, 1e-5


def check_tree(fp, want):
    t = fp.tree()
    codes, fidx, root, left, right, bmin, bsize = want["tree"]
    assert t["n_live"] == codes.size
    assert np.array_equal(t["codes"], codes)
    assert np.array_equal(t["flut_idx"], fidx)
    assert np.array_equal(t["left"], left) and np.array_equal(t["right"], right)
    assert np.array_equal(t["box_min"], bmin) and np.array_equal(t["box_size"], bsize)
    assert np.array_equal(t["rotation_joint"], want["rotation_joint"])


def check_pixels(sc, tables, tree, rj, cam, F, A, D, stride):
    """Oracle render of every `stride`-th pixel of `cam` vs the device maps."""
    R, origin = cam.cam_to_world()
    og, dg, dw = oracle.camera_rays(R, origin, cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                                    cam.height, sc.lo, sc.cell_size)
    pix = np.arange(0, cam.width * cam.height, stride)
    Fo, Ao, Do = oracle.render_rays(*tree, og[pix], dg[pix], dw[pix], 0.0, np.inf,
                                    sc.flut64(), rj, tables.rot_inv, sc.degree, sc.channels,
                                    sc.lambda_th, sc.sigma_dep, True)
    Fg = F.cpu().numpy()[pix].astype(np.float64)
    err = np.abs(Fg - Fo)
    assert err.max() <= F_MAX and err.mean() <= F_MEAN, (err.max(), err.mean())
    assert np.max(np.abs(A.cpu().numpy()[pix] - Ao)) <= 1e-6
    assert np.array_equal(D.cpu().numpy()[pix], Do.astype(np.float32))
    assert (Ao > 0).sum() > 0.05 * pix.size  # the samples actually see the character


def test_configs1_eight_views_one_rebuild():
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c1", frames=1)
    assert len(sc.cameras[0]) == 8 and sc.cameras[0][0].width == 512
    pose = KM.PoseSpec.make(sc.poses[0])
    tables = KM.pose_tables(sc.rig, pose)
    fp = FramePipeline.from_scene(sc)
    views = fp.render_views(pose, sc.cameras[0], lambda_th=sc.lambda_th,
                            sigma_dep=sc.sigma_dep)
    fp.run(pose, sc.cameras[0][0], graph=False, parity=True)  # tree arrays for the check
    fp.stream.synchronize()
    want = oracle.render_frame(sc, tables, sc.cameras[0][0], render=False)
    check_tree(fp, want)
    for v in (0, 3, 6):
        F, A, D = views[v]
        check_pixels(sc, tables, want["tree"], want["rotation_joint"], sc.cameras[0][v], F, A,
                     D, stride=7)
    # a reused-tree view equals a full frame for that camera
    F3, A3, D3 = [x.clone() for x in fp.run(pose, sc.cameras[0][3], graph=False)]
    fp.stream.synchronize()
    assert torch.equal(F3, views[3][0]) and torch.equal(A3, views[3][1])
    assert torch.equal(D3, views[3][2])
    fp.close()


def check_pixels_sliced(sc, tables, tree, rj, cam, F, A, D, stride, width=4):
    """check_pixels for a wide FLUT: the oracle renders `width`-channel
    column slices and each slice is compared with those channels of F."""
    R, origin = cam.cam_to_world()
    og, dg, dw = oracle.camera_rays(R, origin, cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                                    cam.height, sc.lo, sc.cell_size)
    pix = np.arange(0, cam.width * cam.height, stride)
    Fg = F.cpu().numpy()[pix].astype(np.float64)
    H, Ch = (sc.degree + 1) ** 2, sc.channels
    errs = []
    for c0 in range(0, Ch, width):
        cols = [h * Ch + c for h in range(H) for c in range(c0, c0 + width)] + [H * Ch]
        fl = sc.flut32[:, cols].astype(np.float64)
        Fo, Ao, Do = oracle.render_rays(*tree, og[pix], dg[pix], dw[pix], 0.0, np.inf, fl, rj,
                                        tables.rot_inv, sc.degree, width, sc.lambda_th,
                                        sc.sigma_dep, True)
        del fl
        errs.append(np.abs(Fg[:, c0:c0 + width] - Fo))
        if c0 == 0:
            assert np.max(np.abs(A.cpu().numpy()[pix] - Ao)) <= 1e-6
            assert np.array_equal(D.cpu().numpy()[pix], Do.astype(np.float32))
            assert (Ao > 0).sum() > 0.05 * pix.size
    err = np.concatenate(errs, axis=1)
    assert err.max() <= F_MAX and err.mean() <= F_MEAN, (err.max(), err.mean())


def test_configs4_vr_stereo_max_size():
    """configs[4] at full size: 1024^3 grid, ~4 M voxels, C = 32, 32 joints,
    both 1440x1600 eyes of a frame from one rebuild."""
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c4", frames=1)
    assert sc.channels == 32
    assert sc.resolution == 1024 and sc.n_voxels > 3_000_000 and sc.rig.n_joints == 32
    eyes = sc.cameras[0]
    assert len(eyes) == 2 and (eyes[0].width, eyes[0].height) == (1440, 1600)
    pose = KM.PoseSpec.make(sc.poses[0])
    tables = KM.pose_tables(sc.rig, pose)
    fp = FramePipeline.from_scene(sc)
    views = fp.render_views(pose, eyes, lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep)
    fp.run(pose, eyes[0], graph=False, parity=True)
    fp.stream.synchronize()
    # the oracle rebuild only needs the density column
    want = oracle.render_frame(sc, tables, eyes[0], render=False,
                               flut64=sc.flut32[:, -1:].astype(np.float64))
    check_tree(fp, want)
    for e in range(2):
        F, A, D = views[e]
        check_pixels_sliced(sc, tables, want["tree"], want["rotation_joint"], eyes[e], F, A, D,
                            stride=211)
    fp.close()
