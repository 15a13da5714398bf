"""Scene-level drop-ins for the reference's warp / rebuild / render entry
points, computed on the B200.

  warp_voxels         animvox/rigging.py:327-397
  resolve_collisions  animvox/rigging.py:419-459
  build_octree        animvox/volume.py:212-261
  posed_octree        animvox/render.py:154-178
  render_view         animvox/render.py:322-363
  render_frame        animvox/render.py:272-281
  timed_render_frame  animvox/render.py:284-319

They accept the reference's objects (VoxelSet, SkinWeights, Skeleton,
Pose, FLUT, Camera, WarpResult, VoxelOctree) or anything with the same
attributes, and return objects with the reference's field names and dtypes
(the reference's own classes once install.py has run). Host-side work is
what the reference also does on the host and is not on the hot path:
forward kinematics (J joints), argument validation, and the reshape of the
result. Per-frame throughput work lives in frame.FramePipeline.

render_frame / timed_render_frame -- the calls the reference's CLI
(`animate`, `bench`, cli.py:295-416) and WebSocket service
(RenderService.render_png, service.py:121-130) make once per frame -- keep
the character resident on the device between calls: the first call for an
asset builds a FramePipeline (canonical cells, skin weights and the FLUT
uploaded once), later calls only upload the pose tables and camera and run
the device frame (warp -> sort -> resolve -> build -> render) with fp64
alpha/depth maps, exactly the API path's results. A cached pipeline is
dropped when its asset is garbage-collected or its arrays change (data
pointer, shape or a strided content sample).
"""

from __future__ import annotations

import collections
import threading
import time
import weakref

import numpy as np
import torch

from . import _lib
from . import kernels as K
from . import kinematics as KM
from . import types as T
from ._lib import check
from .device import download, empty, ptr, stream_handle, upload
from .errors import ContractViolation, DuplicateMortonError, EmptyWarpError

MAX_GRID_BITS = 21


def _check_resolution(resolution: int) -> None:
    if resolution < 1 or resolution & (resolution - 1):
        raise ContractViolation(f"resolution {resolution} is not a power of two")
    if resolution > (1 << MAX_GRID_BITS):
        raise ContractViolation(f"resolution {resolution} exceeds 2^{MAX_GRID_BITS}")


def _bounds_lo_hi(bounds):
    return np.asarray(bounds.lo, dtype=np.float64), np.asarray(bounds.hi, dtype=np.float64)


def _cell_size(bounds, resolution):
    lo, hi = _bounds_lo_hi(bounds)
    return (hi - lo) / resolution


# ---------------------------------------------------------------------------
# warp


def _key_bits(resolution: int) -> int:
    return 3 * max(1, int(resolution - 1).bit_length())


def _collision_groups_device(d_cells: torch.Tensor, in_bounds: np.ndarray, key_bits: int):
    """rigging.py:373-384: runs of equal live cells among in-bounds voxels,
    members in canonical order, groups in Morton order."""
    ib = np.flatnonzero(in_bounds)
    if ib.size == 0:
        return ()
    L = _lib.lib()
    sel = torch.from_numpy(ib).to(d_cells.device)
    cells64 = d_cells.index_select(0, sel).to(torch.int64).contiguous()
    codes = empty(ib.size, np.uint64)
    check(L.artemis_morton_encode(ptr(cells64), ib.size, ptr(codes), None, stream_handle()),
          "collision groups")
    vals = upload(ib.astype(np.uint32), np.uint32)
    sk, sv = K.sort_pairs_device(codes, vals, key_bits, 8)
    sc = download(sk, np.uint64)
    members = download(sv, np.uint32).astype(np.int64)
    cut = np.flatnonzero(sc[1:] != sc[:-1]) + 1
    starts = np.concatenate([[0], cut])
    ends = np.concatenate([cut, [sc.size]])
    big = (ends - starts) >= 2
    return tuple(members[a:b] for a, b in zip(starts[big], ends[big]))


def warp_voxels(voxels, weights, skeleton, pose):
    """LBS warp of every canonical voxel into `pose` (rigging.py:327-397)."""
    cells = np.ascontiguousarray(voxels.cells, dtype=np.int32)
    n = cells.shape[0]
    jidx = np.ascontiguousarray(weights.joint_indices, dtype=np.int32)
    w = np.ascontiguousarray(weights.weights, dtype=np.float64)
    if jidx.shape[0] != n:
        raise ContractViolation("weights were baked for a different voxel set")
    rig = KM.Rig.from_any(skeleton)
    tables = KM.pose_tables(rig, KM.PoseSpec.from_any(pose))
    res = int(voxels.resolution)
    lo, _ = _bounds_lo_hi(voxels.bounds)
    cell = _cell_size(voxels.bounds, res)
    L = _lib.lib()
    d_cells = upload(cells, np.int32)
    d_j = upload(jidx, np.int32)
    d_w = upload(w, np.float64)
    d_aff = upload(tables.affine34, np.float64)
    pos = empty((n, 3), np.float64)
    out_cells = empty((n, 3), np.int32)
    ib = empty(n, np.uint8)
    rj = empty(n, np.int32)
    lo_h = np.ascontiguousarray(lo, dtype=np.float64)
    cell_h = np.ascontiguousarray(cell, dtype=np.float64)
    check(L.artemis_warp(ptr(d_cells), n, jidx.shape[1], ptr(d_j), ptr(d_w), ptr(d_aff),
                         rig.n_joints, lo_h.ctypes.data, cell_h.ctypes.data, res, ptr(pos),
                         ptr(out_cells), ptr(ib), ptr(rj), stream_handle()), "warp")
    in_bounds = download(ib).astype(bool)
    rotation_joint = download(rj)
    groups = _collision_groups_device(out_cells, in_bounds, _key_bits(res))
    return T.make(
        "WarpResult",
        resolution=res,
        bounds_lo=lo.copy(),
        cell_size=cell,
        positions=download(pos),
        cells=download(out_cells),
        rotations=tables.delta_quats[rotation_joint],
        rotation_joint=rotation_joint,
        joint_rot_inv=tables.rot_inv,
        in_bounds=in_bounds,
        collision_groups=groups,
    )


def identity_warp(voxels):
    """rigging.py:400-416."""
    n = voxels.cells.shape[0]
    rotations = np.zeros((n, 4), dtype=np.float64)
    rotations[:, 0] = 1.0
    lo, _ = _bounds_lo_hi(voxels.bounds)
    centers = lo + (np.asarray(voxels.cells, dtype=np.float64) + 0.5) * \
        _cell_size(voxels.bounds, voxels.resolution)
    return T.make("WarpResult", resolution=voxels.resolution, bounds_lo=lo.copy(),
                  cell_size=_cell_size(voxels.bounds, voxels.resolution), positions=centers,
                  cells=np.asarray(voxels.cells).copy(), rotations=rotations,
                  rotation_joint=np.zeros(n, dtype=np.int32),
                  joint_rot_inv=np.eye(3)[None].copy(), in_bounds=np.ones(n, dtype=bool),
                  collision_groups=())


# ---------------------------------------------------------------------------
# resolve


def resolve_collisions(warp, flut):
    """Winner per live cell + (winner, loser) pairs (rigging.py:419-459)."""
    ib = np.flatnonzero(warp.in_bounds)
    if ib.size == 0:
        return T.make("CollisionResolution", cells=np.empty((0, 3), dtype=np.int32),
                      flut_indices=np.empty(0, dtype=np.int64),
                      pairs=np.empty((0, 2), dtype=np.int64))
    L = _lib.lib()
    cells_ib = np.ascontiguousarray(np.asarray(warp.cells)[ib], dtype=np.int64)
    d_cells = upload(cells_ib, np.int64)
    codes = empty(ib.size, np.uint64)
    check(L.artemis_morton_encode(ptr(d_cells), ib.size, ptr(codes), None, stream_handle()),
          "resolve encode")
    vals = upload(ib.astype(np.uint32), np.uint32)
    sk, sv = K.sort_pairs_device(codes, vals, _key_bits(int(warp.resolution)), 8)
    sigma = upload(np.asarray(flut.densities, dtype=np.float64), np.float64)
    live = empty(ib.size, np.uint64)
    win = empty(ib.size, np.uint32)
    pairs = empty((ib.size, 2), np.int64)
    n_live = empty(1, np.int32)
    ws = K.workspace(L.artemis_resolve_workspace_bytes(ib.size))
    check(L.artemis_resolve_u64(ptr(sk), ptr(sv), ib.size, None, ptr(sigma), ptr(live), ptr(win),
                                ptr(pairs), ptr(n_live), ptr(ws), ws.numel(), stream_handle()),
          "resolve")
    nl = int(download(n_live)[0])
    winners = download(win[:nl], np.uint32).astype(np.int64)
    return T.make("CollisionResolution",
                  cells=np.asarray(warp.cells)[winners].astype(np.int32),
                  flut_indices=winners,
                  pairs=download(pairs[: ib.size - nl]))


# ---------------------------------------------------------------------------
# octree build


def build_octree(voxels, flut_indices=None, *, resolution=None, bounds=None):
    """Morton encode, stable sort, duplicate check, Karras build
    (volume.py:212-261)."""
    if hasattr(voxels, "cells") and hasattr(voxels, "resolution"):
        cells = np.ascontiguousarray(voxels.cells, dtype=np.int32)
        resolution = voxels.resolution
        bounds = voxels.bounds
    else:
        cells = np.ascontiguousarray(np.asarray(voxels), dtype=np.int32)
        if resolution is None or bounds is None:
            raise ContractViolation("raw cell arrays need resolution and bounds")
        _check_resolution(resolution)
    if cells.shape[0] < 1:
        raise ContractViolation("empty cell list")
    if cells.min() < 0 or cells.max() >= resolution:
        raise ContractViolation("cell coordinates outside [0, resolution)")
    n = cells.shape[0]
    if flut_indices is None:
        flut_indices = np.arange(n, dtype=np.uint32)
    else:
        flut_indices = np.ascontiguousarray(np.asarray(flut_indices), dtype=np.uint32)
        if flut_indices.shape != (n,):
            raise ContractViolation("flut_indices length != cell count")
    L = _lib.lib()
    d_cells = upload(cells.astype(np.int64), np.int64)
    codes = empty(n, np.uint64)
    check(L.artemis_morton_encode(ptr(d_cells), n, ptr(codes), None, stream_handle()), "encode")
    sk, sv = K.sort_pairs_device(codes, upload(flut_indices, np.uint32), _key_bits(resolution), 8)
    m = max(n - 1, 1)
    left = empty(m, np.int32)
    right = empty(m, np.int32)
    bmin = empty((m, 3), np.int32)
    bsize = empty((m, 3), np.int32)
    dup = upload(np.array([np.iinfo(np.int32).max], dtype=np.int32), np.int32)
    if n > 1:
        check(L.artemis_build_tree(ptr(sk), n, ptr(left), ptr(right), ptr(bmin), ptr(bsize),
                                   ptr(dup), stream_handle()), "build_tree")
    codes_h = download(sk, np.uint64)
    d = int(download(dup)[0])
    if d != np.iinfo(np.int32).max:
        cell = KM_decode(codes_h[d])
        raise DuplicateMortonError(f"duplicate cell {tuple(int(v) for v in cell)} "
                                   f"(code {int(codes_h[d])})")
    if n == 1:
        root, left_h, right_h = ~0, np.empty(0, np.int32), np.empty(0, np.int32)
        bmin_h, bsize_h = np.empty((0, 3), np.int32), np.empty((0, 3), np.int32)
    else:
        root, left_h, right_h = 0, download(left), download(right)
        bmin_h, bsize_h = download(bmin), download(bsize)
    return T.make("VoxelOctree", resolution=resolution, bounds=bounds, codes=codes_h,
                  flut_idx=download(sv, np.uint32), root=root, left=left_h, right=right_h,
                  box_min=bmin_h, box_size=bsize_h)


def KM_decode(code) -> np.ndarray:
    c = int(code)
    out = []
    for a in range(3):
        v = 0
        for b in range(21):
            v |= ((c >> (3 * b + a)) & 1) << b
        out.append(v)
    return np.array(out, dtype=np.int64)


# ---------------------------------------------------------------------------
# render


def _rotation_tables(warp, n_entries):
    if warp is None:
        return np.zeros(n_entries, dtype=np.int32), np.eye(3)[None].copy()
    return warp.rotation_joint, warp.joint_rot_inv


def render_view(octree, flut, warp, camera, options=None):
    """Integrate every pixel against a posed octree (render.py:322-363)."""
    opts = options or T.RenderOptions()
    cam = KM.PinholeCamera.from_any(camera)
    if getattr(opts, "image_size", None) is not None:
        cam = cam.scaled(*opts.image_size)
    R, origin = cam.cam_to_world()
    lo, _ = _bounds_lo_hi(octree.bounds)
    cell = _cell_size(octree.bounds, octree.resolution)
    og, dg, dw = K.camera_rays_device(R, origin, cam.fx, cam.fy, cam.cx, cam.cy, cam.width,
                                      cam.height, lo, cell)
    rot_index, rot_inv = _rotation_tables(warp, len(flut))
    shade = K.shading_for(flut.data, rot_index, rot_inv, flut.degree, flut.channels)
    tree = K.tree_for(octree.codes, octree.flut_idx, octree.root, octree.left, octree.right,
                      octree.box_min, octree.box_size, shade)
    rays = K.DeviceRays.from_tensors(og, dg, dw, 0.0, np.inf)
    F, A, D = K.render_device(tree, shade, rays, opts.lambda_th, opts.sigma_dep, True)
    h, w = cam.height, cam.width
    return T.make("FrameBuffers",
                  features=download(F).astype(np.float64).reshape(h, w, flut.channels),
                  alpha=download(A).reshape(h, w), depth=download(D).reshape(h, w))


def posed_octree(asset, pose):
    """render.py:154-178."""
    rigged = getattr(asset, "skeleton", None) is not None
    if pose is None or not rigged:
        if pose is not None and not rigged and not _is_canonical(pose):
            raise ContractViolation("asset has no rig; only the canonical pose renders")
        return build_octree(asset.voxels), identity_warp(asset.voxels)
    warp = warp_voxels(asset.voxels, asset.weights, asset.skeleton, pose)
    resolved = resolve_collisions(warp, asset.flut)
    if resolved.cells.shape[0] == 0:
        raise EmptyWarpError(warp.dropped)
    octree = build_octree(resolved.cells, resolved.flut_indices,
                          resolution=asset.voxels.resolution, bounds=asset.voxels.bounds)
    return octree, warp


def _is_canonical(pose) -> bool:
    q = np.asarray(pose.global_rotation)
    return (not np.any(pose.joint_rotations) and q[0] in (1.0, -1.0) and not np.any(q[1:])
            and not np.any(pose.global_translation))


# ---------------------------------------------------------------------------
# persistent device state for the per-frame entry points (CLI, service)


def _array_sig(a) -> tuple:
    """Content key of one asset array: a digest of every byte under the
    default "content" cache policy (an in-place edit, e.g. the reference's
    FLUT.clamp_densities, is a new key), identity only under "identity"
    (kernels.set_cache_policy; the caller then calls DEVICE_ASSETS.clear()
    after editing)."""
    if a is None:
        return (None,)
    return K.content_key(a)


def _asset_sig(asset) -> tuple:
    w = getattr(asset, "weights", None)
    sk = getattr(asset, "skeleton", None)
    return (_array_sig(asset.voxels.cells), _array_sig(asset.flut.data),
            _array_sig(w.joint_indices if w is not None else None),
            _array_sig(w.weights if w is not None else None), id(sk),
            tuple(np.asarray(asset.voxels.bounds.lo, np.float64)),
            tuple(np.asarray(asset.voxels.bounds.hi, np.float64)), int(asset.voxels.resolution))


def _frame_eligible(asset) -> bool:
    r = int(asset.voxels.resolution)
    n = len(asset.voxels.cells)
    sk = getattr(asset, "skeleton", None)
    return (r >= 1 and r & (r - 1) == 0 and r <= (1 << MAX_GRID_BITS) and 0 < n < (1 << 30)
            and (sk is None or len(sk.parents) <= 256) and torch.cuda.is_available())


class _DeviceAssets:
    """LRU of FramePipelines keyed by asset identity + content signature."""

    def __init__(self, capacity: int = 2):
        self.capacity = capacity
        self._d: collections.OrderedDict = collections.OrderedDict()

    def resident(self, asset):
        """(pipeline, signature) cached for this very asset object, without
        digesting its arrays (the caller checks the signature itself), or
        None."""
        ent = self._d.get(id(asset))
        if ent is None or ent[0]() is not asset:
            return None
        return ent[2], ent[1]

    def get(self, asset, sig=None):
        if not _frame_eligible(asset):
            return None
        key = id(asset)
        if sig is None:
            sig = _asset_sig(asset)
        ent = self._d.get(key)
        if ent is not None:
            ref, esig, fp = ent
            if ref() is asset and esig == sig:
                self._d.move_to_end(key)
                return fp
            self._drop(key)
        from .frame import FramePipeline

        fp = FramePipeline.from_asset(asset)
        try:
            ref = weakref.ref(asset, lambda _r, k=key: self._drop(k))
        except TypeError:  # not weak-referenceable: hold it (bounded by capacity)
            ref = (lambda a=asset: a)
        self._d[key] = (ref, sig, fp)
        while len(self._d) > self.capacity:
            self._drop(next(iter(self._d)))
        return fp

    def adopt(self, asset, fp) -> None:
        """Register an already-built pipeline for `asset` (assetio.load_asset:
        the character was decoded straight into device memory)."""
        key = id(asset)
        self._drop(key)
        try:
            ref = weakref.ref(asset, lambda _r, k=key: self._drop(k))
        except TypeError:
            ref = (lambda a=asset: a)
        self._d[key] = (ref, _asset_sig(asset), fp)
        while len(self._d) > self.capacity:
            self._drop(next(iter(self._d)))

    def _drop(self, key):
        ent = self._d.pop(key, None)
        if ent is not None:
            ent[2].close()

    def clear(self):
        for k in list(self._d):
            self._drop(k)


DEVICE_ASSETS = _DeviceAssets()


def _frame_device(asset, pose, camera, opts, timed: bool):
    """One frame through the resident FramePipeline; (FrameBuffers, times).

    Under the "content" cache policy the asset's arrays are digested on every
    call (an in-place edit must take effect, as in the reference, which
    re-reads them per frame). When this asset object already has a resident
    pipeline, the digest runs on a host thread WHILE that pipeline renders
    the frame and reads it out; the frame is returned only if the digest
    equals the resident one, otherwise the pipeline is rebuilt from the new
    content and the frame rendered again -- the result is always that of
    the current content, and the digest's host time overlaps the frame."""
    if K.cache_policy() == "content" and _frame_eligible(asset):
        res = DEVICE_ASSETS.resident(asset)
        if res is not None:
            fp, esig = res
            box = {}

            def digest():
                try:
                    box["sig"] = _asset_sig(asset)
                except BaseException as e:  # re-raised on the calling thread
                    box["err"] = e

            th = threading.Thread(target=digest, name="artemis-asset-digest")
            th.start()
            out = err = None
            try:
                out = _frame_on(fp, asset, pose, camera, opts, timed)
            except Exception as e:  # stale content may be the cause: decided below
                err = e
            finally:
                th.join()
            if "err" in box:
                raise box["err"]
            if box["sig"] == esig:
                if err is not None:
                    raise err
                return out
            fp = DEVICE_ASSETS.get(asset, sig=box["sig"])
            return None if fp is None else _frame_on(fp, asset, pose, camera, opts, timed)
    fp = DEVICE_ASSETS.get(asset)
    if fp is None:
        return None
    return _frame_on(fp, asset, pose, camera, opts, timed)


def _frame_on(fp, asset, pose, camera, opts, timed: bool):
    rigged = getattr(asset, "skeleton", None) is not None
    if pose is not None and not rigged and not _is_canonical(pose):
        raise ContractViolation("asset has no rig; only the canonical pose renders")
    cam = KM.PinholeCamera.from_any(camera)
    if getattr(opts, "image_size", None) is not None:
        cam = cam.scaled(*opts.image_size)
    use_pose = pose if (pose is not None and rigged) else None
    fp.profile(timed)
    F, A, D = fp.run(use_pose, cam, lambda_th=opts.lambda_th, sigma_dep=opts.sigma_dep,
                     graph=not timed, maps64=True)
    stage = fp.stage_ms() if timed else None
    fp.profile(False)
    _, n_live = fp.counts()
    if n_live == 0:
        warp = warp_voxels(asset.voxels, asset.weights, asset.skeleton, pose)
        raise EmptyWarpError(warp.dropped)
    t1 = time.perf_counter()
    features, alpha, depth = fp.host_frame64(F, A, D, cam.width, cam.height)
    frame = T.make("FrameBuffers", features=features, alpha=alpha, depth=depth)
    times = None
    if timed:
        host = time.perf_counter() - t1
        times = {"warp": stage["warp"] / 1e3,
                 "build-octree": (stage["sort"] + stage["resolve"] + stage["build"]) / 1e3,
                 "volume-render": stage["render"] / 1e3 + host}
    return frame, times


def render_frame(asset, pose, camera, options=None):
    """render.py:272-281, on the asset's resident device pipeline."""
    opts = options or T.RenderOptions()
    out = _frame_device(asset, pose, camera, opts, timed=False)
    if out is not None:
        return out[0]
    octree, warp = posed_octree(asset, pose)
    return render_view(octree, asset.flut, warp, camera, opts)


def timed_render_frame(asset, pose, camera, options=None):
    """render_frame plus per-stage seconds keyed like render.py:314-318:
    device time of each stage (CUDA events), the host copy-out and reshape
    counted in "volume-render"."""
    opts = options or T.RenderOptions()
    out = _frame_device(asset, pose, camera, opts, timed=True)
    if out is not None:
        return out
    return _timed_render_frame_api(asset, pose, camera, opts)


def _timed_render_frame_api(asset, pose, camera, options=None):
    """Per-call device path (assets the frame pipeline does not take:
    non-power-of-two grids); each stage synchronised for real device time."""
    opts = options or T.RenderOptions()
    rigged = getattr(asset, "skeleton", None) is not None
    sync = torch.cuda.synchronize
    t0 = time.perf_counter()
    if pose is None or not rigged:
        if pose is not None and not rigged and not _is_canonical(pose):
            raise ContractViolation("asset has no rig; only the canonical pose renders")
        warp = identity_warp(asset.voxels)
        sync()
        t1 = time.perf_counter()
        octree = build_octree(asset.voxels)
    else:
        warp = warp_voxels(asset.voxels, asset.weights, asset.skeleton, pose)
        sync()
        t1 = time.perf_counter()
        resolved = resolve_collisions(warp, asset.flut)
        if resolved.cells.shape[0] == 0:
            raise EmptyWarpError(warp.dropped)
        octree = build_octree(resolved.cells, resolved.flut_indices,
                              resolution=asset.voxels.resolution, bounds=asset.voxels.bounds)
    sync()
    t2 = time.perf_counter()
    frame = render_view(octree, asset.flut, warp, camera, opts)
    sync()
    return frame, {"warp": t1 - t0, "build-octree": t2 - t1,
                   "volume-render": time.perf_counter() - t2}
