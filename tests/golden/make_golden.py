"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package `animvox` from /root/reference/pkg/src with
its compiled backend (`_core`, built by oracle/build_ref.sh into oracle/_ref
and registered as `animvox._core`) and records, on seeded inputs:

* kernels.npz      the flat-array kernel contract on the reference's own
                   test-style inputs (test_backend.py:20-58): Morton
                   encode/decode, sort_order (63-bit and duplicate keys),
                   build_tree (n = 2, 3, 5, 17, 1000 and 20 k cells @512),
                   traverse/forward_fit CSR traces (random, t-range and
                   axis-aligned rays), render_rays (early stop on/off)
* scene_mini.npz   a 64^3 version of configs[0] run end to end through the
                   reference's own rigging/volume/render functions: FK tables,
                   warp_voxels, resolve_collisions, build_octree,
                   rays_for_camera, render_view, forward_fit trace
* backward.npz     backward_rays (training gradients) on the kernel scene's
                   and the 64^3 scene's forward_fit traces, fp64 deterministic
                   and the float32 instantiation
* post.npz         the post-render frame-buffer step (over_background,
                   composite, frame_to_straight_rgba, encode_png) on a seeded
                   3-channel frame
* asset.npz        the .nvo container: digests of save_asset bytes and of
                   load_asset's arrays (rigged and unrigged 64^3 character),
                   and the exception class for each corrupted variant
* fit.npz          the reference's SparseAdam steps, collision-pair term
                   (np.add.at) and L1 sign gradients on seeded inputs
* scaled.npz       the 64^3 scene rendered through render_view with
                   RenderOptions.image_size set (render._scaled_camera,
                   render.py:129-143): the scaled intrinsics, ray directions
                   and the F/A/D maps at 48x40 and 96x80
* scene_c0.npz     configs[0] at full size (128^3, 256^2): SHA-256 digests of
                   every exact array plus a pixel subsample of the maps
* scene_c2.npz     configs[2] at full size (512^3, 1024^2, C = 32 through a
                   duck-typed FLUT, D4): digests plus a pixel subsample

Nothing here is imported by the product; tests read the .npz files only.
"""

from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = os.environ.get("ARTEMIS_REF_ROOT", "/root/reference") + "/pkg/src"


def _import_reference():
    sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
    import _core  # the reference's compiled kernels, built by oracle/build_ref.sh

    sys.modules["animvox._core"] = _core
    os.environ["ANIMVOX_BACKEND"] = "compiled"
    sys.path.insert(0, REF_SRC)
    import animvox.backend as backend

    assert backend.backend_name() == "compiled"
    return backend


backend = _import_reference()
from animvox import _pure  # noqa: E402
from animvox import geometry as G  # noqa: E402
from animvox import render as R  # noqa: E402
from animvox import rigging as RG  # noqa: E402
from animvox import synthetic as SY  # noqa: E402
from animvox import volume as V  # noqa: E402

sys.path.insert(0, REPO)
from paper_2202_05628_b200 import kinematics as K  # noqa: E402
from paper_2202_05628_b200 import synthetic as S  # noqa: E402

kernels = backend.kernels
NT = os.cpu_count() or 1


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a))
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


class DuckFLUT:
    """Bypass FLUT's channels <= 16 check (D4); same attributes."""

    def __init__(self, data, degree, channels):
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        self.degree = degree
        self.channels = channels

    def __len__(self):
        return self.data.shape[0]

    @property
    def densities(self):
        return self.data[:, -1]


# ---------------------------------------------------------------------------
# kernel-contract fixtures (inputs mirror pkg/tests/test_backend.py:20-58)


def _random_tree(rng, res, n):
    cells = np.unique(rng.integers(0, res, size=(n, 3)), axis=0)
    codes = _pure.morton_encode(cells)
    codes = codes[_pure.sort_order(codes)]
    flut_idx = np.arange(codes.size, dtype=np.uint32)
    root, left, right, bmin, bsize = _pure.build_tree(codes)
    return codes, flut_idx, root, left, right, bmin, bsize


def _random_rays(rng, res, count):
    origins = rng.uniform(-0.2 * res, 1.2 * res, size=(count, 3))
    dirs = rng.normal(size=(count, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return origins, dirs


def _random_flut(rng, n, degree, channels):
    h = (degree + 1) * (degree + 1)
    flut = rng.uniform(-0.4, 0.9, size=(n, h * channels + 1))
    flut[:, -1] = rng.uniform(0.0, 40.0, size=n)
    return flut


def _random_rotations(rng, n, n_rot):
    rot_index = rng.integers(0, n_rot, size=n).astype(np.int32)
    mats = []
    for _ in range(n_rot):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        mats.append(G.quat_to_matrix(q).T)
    return rot_index, np.ascontiguousarray(np.stack(mats))


def kernel_fixtures():
    out = {}
    rng = np.random.default_rng(10)
    cells = rng.integers(0, 1 << 21, size=(2000, 3))
    out["morton_cells"] = cells
    out["morton_codes"] = kernels.morton_encode(cells)
    out["morton_decoded"] = kernels.morton_decode(out["morton_codes"])

    rng = np.random.default_rng(11)
    keys = rng.integers(0, 1 << 63, size=20000, dtype=np.int64).astype(np.uint64)
    out["sort63_keys"] = keys
    out["sort63_perm"] = kernels.sort_order(keys, nthreads=NT)
    rng = np.random.default_rng(12)
    dk = rng.integers(0, 50, size=10000, dtype=np.int64).astype(np.uint64)
    out["sortdup_keys"] = dk
    out["sortdup_perm"] = kernels.sort_order(dk, nthreads=NT)
    k30 = np.random.default_rng(13).integers(0, 1 << 30, size=50000).astype(np.uint64)
    out["sort30_keys"] = k30
    out["sort30_perm"] = kernels.sort_order(k30, nthreads=NT)

    for n in (2, 3, 5, 17, 1000):
        rng = np.random.default_rng(n)
        c = np.unique(rng.integers(0, 64, size=(n * 3, 3)), axis=0)[:n]
        codes = _pure.morton_encode(c)
        codes = codes[_pure.sort_order(codes)]
        root, left, right, bmin, bsize = kernels.build_tree(codes, nthreads=NT)
        out[f"tree{n}_codes"] = codes
        out[f"tree{n}_root"] = np.int64(root)
        out[f"tree{n}_left"] = left
        out[f"tree{n}_right"] = right
        out[f"tree{n}_bmin"] = bmin
        out[f"tree{n}_bsize"] = bsize
    rng = np.random.default_rng(99)
    c = np.unique(rng.integers(0, 512, size=(20_000, 3)), axis=0)
    codes = _pure.morton_encode(c)
    codes = codes[_pure.sort_order(codes)]
    root, left, right, bmin, bsize = kernels.build_tree(codes, nthreads=NT)
    out["treeL_codes"] = codes
    out["treeL_root"] = np.int64(root)
    out["treeL_left"] = left
    out["treeL_right"] = right
    out["treeL_bmin"] = bmin
    out["treeL_bsize"] = bsize

    # traversal + render on the test_backend.py "scene" fixture shape
    rng = np.random.default_rng(30)
    tree = _random_tree(rng, 32, 5000)
    nv = tree[0].size
    degree, channels = 2, 3
    flut = _random_flut(rng, nv, degree, channels)
    rot_index, rot_inv = _random_rotations(rng, nv, 6)
    origins, dirs = _random_rays(rng, 32, 400)
    for name, arr in zip(("codes", "flut_idx", "root", "left", "right", "bmin", "bsize"), tree):
        out[f"scene_{name}"] = np.asarray(arr)
    out.update(scene_flut=flut, scene_rot_index=rot_index, scene_rot_inv=rot_inv,
               scene_origins=origins, scene_dirs=dirs)
    args = (*tree, origins, dirs, dirs, 0.0, np.inf, flut, rot_index, rot_inv, degree, channels)
    for es in (False, True):
        f, a, d = kernels.render_rays(*args, 0.01, 5.0, es, NT)
        out[f"scene_F_es{int(es)}"] = f
        out[f"scene_A_es{int(es)}"] = a
        out[f"scene_D_es{int(es)}"] = d
    ff, fa, off, hidx, t0, t1 = kernels.forward_fit(*args, NT)
    out.update(scene_fit_F=ff, scene_fit_A=fa, scene_fit_off=off, scene_fit_idx=hidx,
               scene_fit_t0=t0, scene_fit_t1=t1)
    # t-range and axis-aligned rays (test_backend.py:144-165)
    rng = np.random.default_rng(21)
    tr2 = _random_tree(rng, 16, 800)
    o2, d2 = _random_rays(rng, 16, 200)
    for name, arr in zip(("codes", "flut_idx", "root", "left", "right", "bmin", "bsize"), tr2):
        out[f"tr2_{name}"] = np.asarray(arr)
    f0 = np.zeros((tr2[0].size, 2))
    ri0 = np.zeros(tr2[0].size, dtype=np.int32)
    ro0 = np.eye(3)[None].copy()
    res = kernels.forward_fit(*tr2, o2, d2, d2, 3.0, 11.0, f0, ri0, ro0, 0, 1, NT)
    out.update(tr2_origins=o2, tr2_dirs=d2, tr2_off=res[2], tr2_idx=res[3], tr2_t0=res[4],
               tr2_t1=res[5])
    ax_o, ax_d = [], []
    rng = np.random.default_rng(22)
    for axis in range(3):
        for _ in range(50):
            d = np.zeros(3)
            d[axis] = 1.0 if rng.random() < 0.5 else -1.0
            ax_o.append(rng.uniform(-2, 18, size=3))
            ax_d.append(d)
    ax_o, ax_d = np.array(ax_o), np.array(ax_d)
    res = kernels.forward_fit(*tr2, ax_o, ax_d, ax_d, 0.0, np.inf, f0, ri0, ro0, 0, 1, NT)
    out.update(ax_origins=ax_o, ax_dirs=ax_d, ax_off=res[2], ax_idx=res[3], ax_t0=res[4],
               ax_t1=res[5])
    return out


# ---------------------------------------------------------------------------
# end-to-end scene fixtures through the reference's own entry points


def reference_objects(sc: S.Scene, frame: int = 0):
    bounds = V.Bounds(sc.lo, sc.hi)
    voxels = V.VoxelSet(sc.resolution, bounds, sc.cells)
    data = sc.flut64()
    flut = V.FLUT(data, sc.degree, sc.channels) if sc.channels <= 16 else \
        DuckFLUT(data, sc.degree, sc.channels)
    J = sc.rig.n_joints
    skel = RG.Skeleton(
        names=tuple(f"j{j}" for j in range(J)),
        parents=sc.rig.parents,
        bind_local=tuple(G.RigidTransform(sc.rig.bind_q[j], sc.rig.bind_t[j]) for j in range(J)),
    )
    weights = RG.SkinWeights(sc.skin_idx, sc.skin_w)
    pose = RG.Pose(sc.poses[frame], np.array([1.0, 0.0, 0.0, 0.0]), np.zeros(3))
    return voxels, flut, skel, weights, pose


def reference_camera(cam: K.PinholeCamera):
    return G.Camera(fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=cam.width,
                    height=cam.height,
                    world_to_camera=G.RigidTransform(cam.w2c_q, cam.w2c_t))


def scene_fixture(sc: S.Scene, full: bool, pix_stride: int, fit_rays: int | None):
    out = {}
    timing = {}
    voxels, flut, skel, weights, pose = reference_objects(sc)
    # FK tables as warp_voxels builds them (rigging.py:343-347)
    posed = RG.forward_kinematics(skel, pose)
    deltas = [t.compose(c.invert()) for t, c in zip(posed, skel.canonical_global)]
    out["delta_mats"] = np.stack([d.matrix() for d in deltas])
    out["delta_quats"] = np.stack([d.rotation for d in deltas])
    out["rot_inv"] = np.stack([G.quat_to_matrix(G.quat_conj(d.rotation)) for d in deltas])
    out["pose_wrapped"] = pose.joint_rotations
    # the reference's own orbit camera for the config placement (az 45, el 15)
    cam0 = sc.cameras[0][0]
    rc = SY.orbit_camera(np.radians(45.0), np.radians(15.0), 2.5,
                         image_size=(cam0.width, cam0.height), focal=cam0.fx)
    out["orbit_w2c_q"] = rc.world_to_camera.rotation
    out["orbit_w2c_t"] = rc.world_to_camera.translation

    t = time.perf_counter()
    warp = RG.warp_voxels(voxels, weights, skel, pose)
    timing["warp"] = time.perf_counter() - t
    groups = warp.collision_groups
    g_off = np.zeros(len(groups) + 1, dtype=np.int64)
    g_off[1:] = np.cumsum([g.size for g in groups]) if groups else []
    g_mem = np.concatenate(groups) if groups else np.zeros(0, dtype=np.int64)
    t = time.perf_counter()
    resolved = RG.resolve_collisions(warp, flut)
    timing["resolve"] = time.perf_counter() - t
    t = time.perf_counter()
    octree = V.build_octree(resolved.cells, resolved.flut_indices,
                            resolution=voxels.resolution, bounds=voxels.bounds)
    timing["build"] = time.perf_counter() - t
    cam = sc.cameras[0][0]
    rcam = reference_camera(cam)
    origins, dirs = G.rays_for_camera(rcam)
    opts = R.RenderOptions(lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep)
    t = time.perf_counter()
    frame = R.render_view(octree, flut, warp, rcam, opts)
    timing["render"] = time.perf_counter() - t

    exact = {
        "warp_positions": warp.positions, "warp_cells": warp.cells,
        "warp_in_bounds": warp.in_bounds, "warp_rotation_joint": warp.rotation_joint,
        "warp_rotations": warp.rotations, "groups_off": g_off, "groups_mem": g_mem,
        "res_cells": resolved.cells, "res_flut": resolved.flut_indices,
        "res_pairs": resolved.pairs, "oct_codes": octree.codes, "oct_flut": octree.flut_idx,
        "oct_left": octree.left, "oct_right": octree.right, "oct_bmin": octree.box_min,
        "oct_bsize": octree.box_size, "rays_o": origins, "rays_d": dirs,
        "depth": frame.depth,
    }
    out["oct_root"] = np.int64(octree.root)
    if full:
        out.update(exact)
        out["F"] = frame.features
        out["A"] = frame.alpha
    for k, v in exact.items():
        out[f"sha_{k}"] = np.array(digest(v))
    # pixel subsample of the tolerance maps (row-major pixel ids)
    npix = cam.width * cam.height
    pix = np.arange(0, npix, pix_stride)
    out["sub_pix"] = pix
    out["sub_F"] = frame.features.reshape(npix, -1)[pix]
    out["sub_A"] = frame.alpha.reshape(-1)[pix]
    out["sub_D"] = frame.depth.reshape(-1)[pix]
    out["stat_F_absmean"] = np.float64(np.abs(frame.features).mean())
    out["stat_A_sum"] = np.float64(frame.alpha.sum())
    # CSR hit trace (forward_fit) over all rays or a prefix subset
    cell = octree.cell_size
    sel = slice(None) if fit_rays is None else slice(0, fit_rays)
    og = np.ascontiguousarray((origins[sel] - octree.bounds.lo) / cell)
    dg = np.ascontiguousarray(dirs[sel] / cell)
    rot_index, rot_inv = warp.rotation_joint, warp.joint_rot_inv
    t = time.perf_counter()
    ff, fa, off, hidx, t0, t1 = kernels.forward_fit(
        octree.codes, octree.flut_idx, octree.root, octree.left, octree.right,
        octree.box_min, octree.box_size, og, dg, np.ascontiguousarray(dirs[sel]), 0.0,
        np.inf, flut.data, rot_index, rot_inv, flut.degree, flut.channels, NT)
    timing["forward_fit"] = time.perf_counter() - t
    trace = {"fit_off": off, "fit_idx": hidx, "fit_t0": t0, "fit_t1": t1}
    for k, v in trace.items():
        out[f"sha_{k}"] = np.array(digest(v))
    if full:
        out.update(trace)
    out["fit_rays"] = np.int64(og.shape[0])
    out["n_hits"] = np.int64(hidx.size)
    out["n_leaves"] = np.int64(octree.codes.size)
    out["n_inbounds"] = np.int64(warp.in_bounds.sum())
    meta = dict(timing=timing, numpy=np.__version__, machine=platform.machine(),
                processor=platform.processor(), threads=NT)
    out["meta"] = np.array(json.dumps(meta))
    return out


def backward_fixtures():
    """backward_rays (_core.pyx:661-755) on two traced batches: the
    test_backend-style kernel scene (degree 2, C = 3, normal dL/dF, dL/dA as
    in test_backend.py:201-216) and the 64^3 posed scene's forward_fit
    trace (degree 2, C = 16, sign-style losses as fit.py:486-488 feeds it).
    Deterministic fp64 and the float32 instantiation."""
    from animvox import _core

    out = {}
    k = np.load(os.path.join(HERE, "kernels.npz"))
    rng = np.random.default_rng(31)
    n = k["scene_origins"].shape[0]
    dldf = rng.normal(size=(n, 3))
    dlda = rng.normal(size=n)
    common = (k["scene_fit_off"], k["scene_fit_idx"], k["scene_fit_t0"], k["scene_fit_t1"],
              k["scene_dirs"], k["scene_rot_index"], k["scene_rot_inv"])
    g64 = _core.backward_rays(*common, k["scene_flut"], dldf, dlda, 2, 3, True, 1)
    gp = _pure.backward_rays(*common, k["scene_flut"], dldf, dlda, 2, 3)
    assert np.array_equal(np.asarray(g64), gp)
    g32 = _core.backward_rays(*common, np.ascontiguousarray(k["scene_flut"], dtype=np.float32),
                              dldf.astype(np.float32), dlda.astype(np.float32), 2, 3, True, 1)
    out.update(k_dldf=dldf, k_dlda=dlda, k_grad64=np.asarray(g64), k_grad32=np.asarray(g32))

    m = np.load(os.path.join(HERE, "scene_mini.npz"))
    sc = S.make_scene("c0", resolution=64, image=(64, 64))
    n = int(m["fit_rays"])
    rng = np.random.default_rng(41)
    dldf = np.sign(rng.normal(size=(n, sc.channels))) / n
    dlda = np.sign(rng.normal(size=n)) / n
    common = (m["fit_off"], m["fit_idx"], m["fit_t0"], m["fit_t1"], m["rays_d"],
              m["warp_rotation_joint"], m["rot_inv"])
    g64 = _core.backward_rays(*common, sc.flut64(), dldf, dlda, sc.degree, sc.channels, True, 1)
    g32 = _core.backward_rays(*common, np.ascontiguousarray(sc.flut32), dldf.astype(np.float32),
                              dlda.astype(np.float32), sc.degree, sc.channels, True, 1)
    out.update(m_dldf=dldf, m_dlda=dlda, m_grad64=np.asarray(g64), m_grad32=np.asarray(g32))
    return out


def post_fixtures():
    """The post-render frame-buffer step through the reference's own code
    (render.py:98-104 over_background, :366-382 composite, assetio.py:265-275
    frame_to_straight_rgba, :232-245 encode_png decoded back to uint8) on a
    seeded 3-channel frame: fp32-representable premultiplied F, alpha with
    exact zeros and values above the features (clip), depth with +inf, a
    background depth with ties, +inf and nearer/farther pixels."""
    import io

    from PIL import Image

    from animvox import assetio as AIO

    rng = np.random.default_rng(77)
    h, w = 24, 20
    a = rng.uniform(0.0, 1.0, size=(h, w))
    a[rng.uniform(size=(h, w)) < 0.25] = 0.0
    a = a.astype(np.float32).astype(np.float64)
    f = (rng.uniform(-0.1, 1.3, size=(h, w, 3)) * a[:, :, None]).astype(np.float32)
    f = f.astype(np.float64)
    d = rng.uniform(1.0, 3.0, size=(h, w)).astype(np.float32).astype(np.float64)
    d[a == 0.0] = np.inf
    bgc = rng.uniform(0.0, 1.0, size=(h, w, 3))
    bgd = rng.uniform(1.0, 3.0, size=(h, w))
    bgd[::5, ::3] = d[::5, ::3]  # ties go to the volume (<=)
    bgd[1::7, :] = np.inf
    color = np.array([0.2, 0.5, 0.9])
    fb = R.FrameBuffers(features=f, alpha=a, depth=d)
    over = fb.over_background(color)
    comp = R.composite(fb, bgc, bgd)
    rgba = AIO.frame_to_straight_rgba(f, a)
    png = AIO.encode_png(rgba)
    q = np.asarray(Image.open(io.BytesIO(png)).convert("RGBA"))
    return dict(F=f, A=a, D=d, bg_color=bgc, bg_depth=bgd, color=color, over=over,
                composite=comp, rgba=rgba, rgba8=q)


def asset_fixtures():
    """The .nvo container (assetio.py:49-202) through the reference: SHA-256
    of save_asset's bytes and of every array load_asset returns, for a rigged
    64^3 character (C = 16) and an unrigged one; and the exception class
    load_asset raises for each corruption of the rigged file."""
    from animvox import assetio as AIO

    out = {}
    sc = S.make_scene("c0", resolution=64, image=(64, 64))
    voxels, flut, skel, weights, _ = reference_objects(sc)
    cases = {"rig": R.CharacterAsset(voxels, flut, skel, weights),
             "still": R.CharacterAsset(voxels, flut)}
    for name, asset in cases.items():
        data = AIO.save_asset(asset)
        back = AIO.load_asset(data)
        out[f"{name}_sha_bytes"] = np.array(hashlib.sha256(data).hexdigest())
        out[f"{name}_size"] = np.int64(len(data))
        arrs = {"cells": back.voxels.cells, "flut": back.flut.data,
                "lo": back.voxels.bounds.lo, "hi": back.voxels.bounds.hi}
        if back.skeleton is not None:
            arrs.update(parents=back.skeleton.parents,
                        bind=np.array([[*b.rotation, *b.translation]
                                       for b in back.skeleton.bind_local]),
                        joint_idx=back.weights.joint_indices, weights=back.weights.weights)
            out[f"{name}_names"] = np.array("|".join(back.skeleton.names))
        for k, v in arrs.items():
            out[f"{name}_sha_{k}"] = np.array(digest(v))
        out[f"{name}_resolution"] = np.int64(back.voxels.resolution)
    data = AIO.save_asset(cases["rig"])
    hs = 54
    n = len(voxels)
    width = flut.data.shape[1]
    flut_end = hs + 12 * n + 4 * width * n
    bad = bytearray(data)
    bad[hs + 8:hs + 12] = bad[hs + 20:hs + 24]  # two leaves share a FLUT row
    corrupt = {
        "short_header": data[:40], "magic": b"NVO2" + data[4:],
        "version": data[:4] + (2).to_bytes(4, "little") + data[8:],
        "zero_count": data[:12] + (0).to_bytes(8, "little") + data[20:],
        "short_leaves": data[:hs + 12 * (n // 2)], "short_flut": data[:flut_end - 3],
        "not_permutation": bytes(bad),
        "rig_offset": data[:46] + (flut_end + 1).to_bytes(8, "little") + data[54:],
        "short_rig": data[:-2], "trailing": data + b"\0",
    }
    for k, v in corrupt.items():
        try:
            AIO.load_asset(v)
            out[f"err_{k}"] = np.array("none")
        except Exception as exc:  # the reference's class name is the fixture
            out[f"err_{k}"] = np.array(type(exc).__name__)
    return out


def fit_fixtures():
    """The reference's own training bookkeeping on seeded inputs: three
    SparseAdam steps (fit.py:308-330) with FLUT.clamp_densities, the
    collision-pair term through GradBuffer.add (np.add.at, repeated rows)
    and the L1 sign gradients of fit.py:486-488."""
    from animvox import fit as FIT

    rng = np.random.default_rng(123)
    n, width = 40, 28
    params = rng.uniform(-1, 1, size=(n, width))
    params[:, -1] = rng.uniform(0.0, 0.02, size=n)
    cfg = FIT.FitConfig(learning_rate=0.05)
    opt = FIT.SparseAdam(params.shape, cfg)
    grads, touches = [], []
    p = params.copy()
    for step in range(3):
        g = np.zeros_like(p)
        touched = rng.uniform(size=n) < 0.5
        g[touched] = rng.normal(size=(int(touched.sum()), width))
        g[touched, -1] = np.abs(g[touched, -1]) * 5  # drive densities below zero
        grads.append(g)
        touches.append(touched)
        opt.step(p, FIT.GradBuffer(values=g.copy(), touched=touched.copy()))
        fl = V.FLUT.__new__(V.FLUT)
        fl.data = p
        V.FLUT.clamp_densities(fl)
    pairs = rng.integers(0, n, size=(60, 2))
    pairs[:10, 0] = 3  # repeated winners
    gbuf = FIT.GradBuffer(values=np.zeros((n, width)), touched=np.zeros(n, bool))
    s = np.sign(params[pairs[:, 0]] - params[pairs[:, 1]])
    s *= 0.01 / (pairs.shape[0] * width)
    gbuf.add(pairs[:, 0], s)
    gbuf.add(pairs[:, 1], -s)
    F = rng.normal(size=(50, 3)).astype(np.float32)
    A = rng.uniform(size=50)
    gt_f = np.where(rng.uniform(size=(50, 3)) < 0.2, F.astype(np.float64), rng.normal(size=(50, 3)))
    gt_a = np.where(rng.uniform(size=50) < 0.2, A, rng.uniform(size=50))
    n_p = 50
    return dict(params0=params, grads=np.stack(grads), touches=np.stack(touches), params3=p,
                m3=opt.m, v3=opt.v, pairs=pairs, vrt_grad=gbuf.values, vrt_touched=gbuf.touched,
                F=F, A=A, gt_f=gt_f, gt_a=gt_a,
                dldf=np.sign(F.astype(np.float64) - gt_f) / n_p,
                dlda=np.sign(A - gt_a) / n_p,
                loss=np.float64(FIT.loss_rgba(F, A, gt_f, gt_a)))


def scaled_fixtures():
    """render_view with opts.image_size (render.py:129-143, 322-363) on the
    64^3 scene: the camera the reference derives and the maps it renders, at a
    size below and a size above the camera's own 64x64 (non-square both)."""
    sc = S.make_scene("c0", resolution=64, image=(64, 64))
    voxels, flut, skel, weights, pose = reference_objects(sc)
    warp = RG.warp_voxels(voxels, weights, skel, pose)
    resolved = RG.resolve_collisions(warp, flut)
    octree = V.build_octree(resolved.cells, resolved.flut_indices,
                            resolution=voxels.resolution, bounds=voxels.bounds)
    rcam = reference_camera(sc.cameras[0][0])
    out = {"sizes": np.array([[48, 40], [96, 80]], dtype=np.int64)}
    for i, (w, h) in enumerate(out["sizes"].tolist()):
        cam = R._scaled_camera(rcam, (w, h))
        out[f"intr{i}"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy], dtype=np.float64)
        out[f"wh{i}"] = np.array([cam.width, cam.height], dtype=np.int64)
        _, dirs = G.rays_for_camera(cam)
        out[f"sha_rays_d{i}"] = np.array(digest(dirs))
        opts = R.RenderOptions(lambda_th=sc.lambda_th, sigma_dep=sc.sigma_dep,
                               image_size=(w, h))
        frame = R.render_view(octree, flut, warp, rcam, opts)
        out[f"F{i}"] = frame.features
        out[f"A{i}"] = frame.alpha
        out[f"D{i}"] = frame.depth
    return out


def main(which):
    t = time.time()
    if "scaled" in which:
        np.savez_compressed(os.path.join(HERE, "scaled.npz"), **scaled_fixtures())
        print("scaled.npz", time.time() - t)
    if "kernels" in which:
        np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kernel_fixtures())
        print("kernels.npz", time.time() - t)
    if "mini" in which:
        sc = S.make_scene("c0", resolution=64, image=(64, 64))
        np.savez_compressed(os.path.join(HERE, "scene_mini.npz"),
                            **scene_fixture(sc, full=True, pix_stride=1, fit_rays=None))
        print("scene_mini.npz", sc.n_voxels, time.time() - t)
    if "backward" in which:
        np.savez_compressed(os.path.join(HERE, "backward.npz"), **backward_fixtures())
        print("backward.npz", time.time() - t)
    if "post" in which:
        np.savez_compressed(os.path.join(HERE, "post.npz"), **post_fixtures())
        print("post.npz", time.time() - t)
    if "asset" in which:
        np.savez_compressed(os.path.join(HERE, "asset.npz"), **asset_fixtures())
        print("asset.npz", time.time() - t)
    if "fit" in which:
        np.savez_compressed(os.path.join(HERE, "fit.npz"), **fit_fixtures())
        print("fit.npz", time.time() - t)
    if "c0" in which:
        sc = S.make_scene("c0")
        np.savez_compressed(os.path.join(HERE, "scene_c0.npz"),
                            **scene_fixture(sc, full=False, pix_stride=7, fit_rays=None))
        print("scene_c0.npz", sc.n_voxels, time.time() - t)
    if "c2" in which:
        sc = S.make_scene("c2")
        np.savez_compressed(os.path.join(HERE, "scene_c2.npz"),
                            **scene_fixture(sc, full=False, pix_stride=97, fit_rays=None))
        print("scene_c2.npz", sc.n_voxels, time.time() - t)


if __name__ == "__main__":
    main(sys.argv[1:] or ["kernels", "mini", "backward", "post", "asset", "fit", "scaled", "c0", "c2"])
