"""The reference's flat-array kernel contract, on the B200.

A module with the same names, argument meanings, dtypes and error
behaviour as ``animvox._core`` / ``animvox._pure`` (selected by
animvox/backend.py:19-31), so it can be bound as ``animvox.backend.kernels``
(see install.py). Every call moves its numpy arguments to the device, runs
the libartemis kernel through the C ABI and returns freshly allocated numpy
arrays in the reference's dtypes:

  morton_encode  _core.pyx:79-92     morton_decode  :95-105
  sort_order     :111-167            build_tree     :193-246
  traverse_ray   :358-389            render_rays    :473-559
  forward_fit    :562-655

``nthreads`` is accepted and ignored (results never depended on it).
  backward_rays  :661-755 (training gradients)
"""

from __future__ import annotations

import collections
import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from ._lib import check
from .device import device, download, empty, ptr, stream_handle, upload, workspace

IS_COMPILED = True
BACKEND = "artemis-b200"

_MORTON_LIMIT = 1 << 21


def morton_encode(coords):
    arr = np.ascontiguousarray(coords, dtype=np.int64)
    if arr.size and (arr.min() < 0 or arr.max() >= _MORTON_LIMIT):
        raise ValueError("grid coordinates outside [0, 2^21)")
    arr = arr.reshape(-1, 3)
    n = arr.shape[0]
    if n == 0:
        return np.empty(0, dtype=np.uint64)
    L = _lib.lib()
    d_in = upload(arr, np.int64)
    d_out = empty(n, np.uint64)
    check(L.artemis_morton_encode(ptr(d_in), n, ptr(d_out), None, stream_handle()),
          "morton_encode")
    return download(d_out, np.uint64)


def morton_decode(codes):
    c = np.ascontiguousarray(codes, dtype=np.uint64).reshape(-1)
    n = c.size
    if n == 0:
        return np.empty((0, 3), dtype=np.int64)
    L = _lib.lib()
    d_in = upload(c, np.uint64)
    d_out = empty((n, 3), np.int64)
    check(L.artemis_morton_decode(ptr(d_in), n, ptr(d_out), stream_handle()), "morton_decode")
    return download(d_out)


def sort_pairs_device(keys: torch.Tensor, vals: torch.Tensor | None, key_bits: int,
                      key_bytes: int):
    """Stable device sort of (key, value); returns (sorted keys, values)."""
    L = _lib.lib()
    n = keys.numel()
    ws = workspace(L.artemis_sort_workspace_bytes(n, key_bits, key_bytes))
    k_out = torch.empty_like(keys)
    v_out = torch.empty(n, dtype=torch.int32, device=keys.device)
    fn = L.artemis_sort_pairs_u32 if key_bytes == 4 else L.artemis_sort_pairs_u64
    check(fn(ptr(keys), ptr(vals), ptr(k_out), ptr(v_out), n, key_bits, ptr(ws), ws.numel(),
             stream_handle()), "sort")
    return k_out, v_out


def sort_order(codes, nthreads=1):
    c = np.ascontiguousarray(codes, dtype=np.uint64).reshape(-1)
    n = c.size
    if n <= 1:
        return np.arange(n, dtype=np.int64)
    bits = max(1, int(c.max()).bit_length())
    if bits <= 32:
        keys = upload(c.astype(np.uint32), np.uint32)
        _, perm = sort_pairs_device(keys, None, bits, 4)
    else:
        keys = upload(c, np.uint64)
        _, perm = sort_pairs_device(keys, None, bits, 8)
    return download(perm).astype(np.int64)


def build_tree(codes, nthreads=1):
    c = np.ascontiguousarray(codes, dtype=np.uint64).reshape(-1)
    n = c.size
    if n == 0:
        raise ValueError("empty leaf set")
    m = max(n - 1, 1)
    if n == 1:
        return (~0, np.empty(0, np.int32), np.empty(0, np.int32), np.empty((0, 3), np.int32),
                np.empty((0, 3), np.int32))
    L = _lib.lib()
    d_c = upload(c, np.uint64)
    left = empty(m, np.int32)
    right = empty(m, np.int32)
    bmin = empty((m, 3), np.int32)
    bsize = empty((m, 3), np.int32)
    check(L.artemis_build_tree(ptr(d_c), n, ptr(left), ptr(right), ptr(bmin), ptr(bsize), None,
                               stream_handle()), "build_tree")
    return 0, download(left), download(right), download(bmin), download(bsize)


def morton_decode_host_all(codes) -> np.ndarray:
    """Vectorised host decode (x lowest slot, 21 bits per axis)."""
    c = np.asarray(codes, dtype=np.uint64)
    out = np.zeros((c.size, 3), dtype=np.int64)
    for a in range(3):
        v = np.zeros(c.size, dtype=np.uint64)
        for b in range(21):
            v |= ((c >> np.uint64(3 * b + a)) & np.uint64(1)) << np.uint64(b)
        out[:, a] = v.astype(np.int64)
    return out


def morton_decode_host(codes) -> np.ndarray:
    """Host decode of a few codes (no device needed)."""
    out = np.zeros((len(codes), 3), dtype=np.int64)
    for i, c in enumerate(np.asarray(codes, dtype=np.uint64)):
        c = int(c)
        for a in range(3):
            out[i, a] = sum(((c >> (3 * b + a)) & 1) << b for b in range(21))
    return out


class DeviceTree:
    """A reference-layout tree on the device plus its packed traversal copy
    (leaf records carry density and rotation index when `shade` is given)."""

    def __init__(self, codes, flut_idx, root, left, right, box_min, box_size, shade=None):
        c = np.ascontiguousarray(codes, dtype=np.uint64).reshape(-1)
        n = c.size
        if n < 1:
            raise ValueError("empty leaf set")
        L = _lib.lib()
        self.n = n
        self.codes = upload(c, np.uint64)
        self.flut_idx = upload(np.asarray(flut_idx).reshape(-1), np.uint32)
        self.h2d_bytes = c.nbytes + 4 * n
        if n > 1:
            self.left = upload(left, np.int32)
            self.right = upload(right, np.int32)
            self.bmin = upload(np.asarray(box_min).reshape(-1, 3), np.int32)
            self.bsize = upload(np.asarray(box_size).reshape(-1, 3), np.int32)
            self.h2d_bytes += 32 * (n - 1)
        else:
            self.left = self.right = self.bmin = self.bsize = None
        self.nodes = workspace(64 * n)
        self.leaves = workspace(32 * n)
        sig = shade.sigma if shade is not None else None
        rix = shade.rot_index if shade is not None else None
        check(L.artemis_pack_tree(ptr(self.codes), ptr(self.flut_idx), n, int(root),
                                  ptr(self.left), ptr(self.right), ptr(self.bmin), ptr(self.bsize),
                                  ptr(sig), ptr(rix), ptr(self.nodes), ptr(self.leaves),
                                  stream_handle()), "pack_tree")
        # leaf-cell bounds, decoded on the device (no host pass over the codes)
        xyz = empty((n, 3), np.int64)
        check(L.artemis_morton_decode(ptr(self.codes), n, ptr(xyz), stream_handle()),
              "morton_decode")
        ext = torch.stack([xyz.min(dim=0).values, xyz.max(dim=0).values]).cpu().numpy()
        del xyz
        if n > 1:
            bm = np.asarray(box_min).reshape(-1, 3)
            bs = np.asarray(box_size).reshape(-1, 3)
            r = int(root) if int(root) >= 0 else 0
            cmax = float((bm[r] + bs[r]).max())
        else:
            cmax = float(ext[1].max() + 1)
        self.bmap = None
        self._bricks(L, ext)
        self.view = _lib.TreeView(ptr(self.nodes), ptr(self.leaves), n, None, cmax,
                                  C.pointer(self.bmap) if self.bmap is not None else None)

    MAX_BRICK_TABLE = 1 << 24  # entries (64 MB): beyond that the tree DFS is used

    def _bricks(self, L, ext):
        """Occupancy brick map over the leaves' brick-coordinate box, when it
        is small enough for a dense table (same results either way)."""
        lo = ext[0] >> 3
        hi = ext[1] >> 3
        dims = (hi - lo + 1).astype(np.int32)
        if int(np.prod(dims.astype(np.int64))) > self.MAX_BRICK_TABLE:
            return
        org = np.ascontiguousarray(lo.astype(np.int32))
        dims = np.ascontiguousarray(dims)
        self.bstore = workspace(L.artemis_brickmap_bytes(self.n, dims.ctypes.data))
        bm = _lib.BrickMap()
        check(L.artemis_brickmap_build(ptr(self.codes), self.n, org.ctypes.data, dims.ctypes.data,
                                       ptr(self.bstore), self.bstore.numel(), C.byref(bm),
                                       stream_handle()), "brickmap")
        self.bmap = bm


UPLOAD_CHUNK_BYTES = 32 << 20  # pinned staging chunk of the FLUT upload


class DeviceShading:
    """FLUT split into fp32 coefficients + fp64 density, rotation tables.

    The FLUT crosses PCIe in pinned chunks, each split on the device as it
    lands (double-buffered), so no FLUT-sized staging copy exists on either
    side."""

    def __init__(self, flut, rot_index, rot_inv, degree, channels):
        L = _lib.lib()
        fl = np.asarray(flut)
        if fl.ndim != 2:
            raise ValueError("flut must be (N, H*C+1)")
        if fl.dtype not in (np.float32, np.float64):
            fl = fl.astype(np.float64)
        n, width = fl.shape
        self.coef = empty((n, max(width - 1, 1)), np.float32)
        self.sigma = empty(n, np.float64)
        self._upload_split(L, fl)
        self.rot_index = upload(np.asarray(rot_index).reshape(-1), np.int32)
        self.rot_inv = upload(np.asarray(rot_inv).reshape(-1, 9), np.float64)
        self.h2d_bytes = fl.nbytes + 4 * self.rot_index.numel() + 8 * self.rot_inv.numel()
        self.view = _lib.Shading(ptr(self.coef), ptr(self.sigma), ptr(self.rot_index),
                                 ptr(self.rot_inv), int(degree), int(channels), width - 1)

    def _upload_split(self, L, fl):
        n, width = fl.shape
        if n == 0:
            return
        split = L.artemis_flut_split_f32 if fl.dtype == np.float32 else L.artemis_flut_split_f64
        tdt = torch.float32 if fl.dtype == np.float32 else torch.float64
        rows = max(1, UPLOAD_CHUNK_BYTES // (width * fl.itemsize))
        if rows >= n:  # small table: one plain copy
            d_fl = upload(fl, fl.dtype)
            check(split(ptr(d_fl), n, width, ptr(self.coef), ptr(self.sigma), stream_handle()),
                  "flut_split")
            return
        st = torch.cuda.current_stream()
        host = [torch.empty(rows * width, dtype=tdt, pin_memory=True) for _ in range(2)]
        dev = [torch.empty(rows * width, dtype=tdt, device=device()) for _ in range(2)]
        done = [None, None]
        hc = max(width - 1, 1)
        for i, r0 in enumerate(range(0, n, rows)):
            b = i & 1
            cnt = min(rows, n - r0)
            if done[b] is not None:
                done[b].synchronize()  # the copy out of host[b] has finished
            hb = host[b].numpy()[:cnt * width]
            np.copyto(hb.reshape(cnt, width), fl[r0:r0 + cnt])
            dev[b][:cnt * width].copy_(host[b][:cnt * width], non_blocking=True)
            check(split(ptr(dev[b]), cnt, width, self.coef.data_ptr() + 4 * hc * r0,
                        self.sigma.data_ptr() + 8 * r0, stream_handle()), "flut_split")
            done[b] = torch.cuda.Event()
            done[b].record(st)
        st.synchronize()


# ---------------------------------------------------------------------------
# device cache of the kernel-contract shim ("device-cached
# tree and FLUT keyed by array identity plus a content check, no per-call
# re-upload"). The reference re-reads its arguments on every call, so the
# key is the FULL content of each array (128-bit digest of every byte,
# artemis_host_checksum): an in-place edit of the FLUT between two calls is
# a new key. Policy "identity" skips the digest (address, shape, dtype,
# strides only) for callers that promise immutability or call
# invalidate_cache() after editing.

_POLICY = os.environ.get("ARTEMIS_CACHE_POLICY", "content")
_HASH_THREADS = max(1, min(16, os.cpu_count() or 1))
_STATS = {"hits": 0, "misses": 0, "h2d_bytes": 0, "hash_bytes": 0}
_SHADE_CACHE: "collections.OrderedDict" = collections.OrderedDict()
_TREE_CACHE: "collections.OrderedDict" = collections.OrderedDict()
SHADE_CAPACITY = 2
TREE_CAPACITY = 4


def set_cache_policy(policy: str) -> None:
    """"content" (default): device copies keyed by a digest of every byte;
    "identity": by address/shape/dtype/strides only (the caller invalidates)."""
    global _POLICY
    if policy not in ("content", "identity"):
        raise ValueError("cache policy must be 'content' or 'identity'")
    _POLICY = policy
    invalidate_cache()


def cache_policy() -> str:
    """The current cache policy ("content" or "identity")."""
    return _POLICY


def invalidate_cache() -> None:
    """Drop every cached device FLUT / tree (after in-place edits under the
    "identity" policy; harmless otherwise)."""
    _SHADE_CACHE.clear()
    _TREE_CACHE.clear()


def cache_stats(reset: bool = False) -> dict:
    out = dict(_STATS, policy=_POLICY, shadings=len(_SHADE_CACHE), trees=len(_TREE_CACHE))
    if reset:
        for k in _STATS:
            _STATS[k] = 0
    return out


def content_key(a, dtype=None) -> tuple:
    """Cache key of one argument array as the kernels will see it."""
    arr = np.asarray(a) if dtype is None else np.asarray(a, dtype=dtype)
    if _POLICY == "identity":
        return ("id", arr.__array_interface__["data"][0], arr.shape, str(arr.dtype), arr.strides)
    arr = np.ascontiguousarray(arr)
    out = (C.c_uint64 * 2)()
    check(_lib.load_library().artemis_host_checksum(arr.ctypes.data, arr.nbytes, _HASH_THREADS,
                                                    out), "checksum")
    _STATS["hash_bytes"] += arr.nbytes
    return (arr.shape, str(arr.dtype), int(out[0]), int(out[1]))


def _lru_get(cache, key, capacity, make, on_evict=None):
    ent = cache.get(key)
    if ent is not None:
        cache.move_to_end(key)
        _STATS["hits"] += 1
        return ent
    _STATS["misses"] += 1
    while len(cache) >= capacity:
        old, _ = cache.popitem(last=False)
        if on_evict is not None:
            on_evict(old)
    ent = make()
    _STATS["h2d_bytes"] += getattr(ent, "h2d_bytes", 0)
    cache[key] = ent
    return ent


def shading_for(flut, rot_index, rot_inv, degree, channels):
    """Cached DeviceShading of (flut, rotation tables)."""
    fl = np.asarray(flut)
    if fl.dtype not in (np.float32, np.float64):
        fl = fl.astype(np.float64)
    key = (content_key(fl), content_key(rot_index, np.int32), content_key(rot_inv, np.float64),
           int(degree), int(channels))
    sh = _lru_get(_SHADE_CACHE, key, SHADE_CAPACITY,
                  lambda: DeviceShading(fl, rot_index, rot_inv, degree, channels),
                  on_evict=_drop_trees_of)
    sh.key = key
    return sh


def _drop_trees_of(shade_key) -> None:
    """Trees embed their shading's density/rotation (and keep it alive):
    they leave the cache with it."""
    for k in [k for k in _TREE_CACHE if k[1] == shade_key]:
        del _TREE_CACHE[k]


def tree_for(codes, flut_idx, root, left, right, box_min, box_size, shade, any_shade=False):
    """Cached DeviceTree (packed nodes, leaf records, brick map) of a
    reference-layout tree; leaf records embed `shade`'s density/rotation.
    any_shade: a traversal-only caller takes a cached tree of the same
    arrays built for any shading (the walk never reads those fields)."""
    tkey = (content_key(codes, np.uint64), content_key(flut_idx, np.uint32), int(root),
            content_key(left, np.int32), content_key(right, np.int32),
            content_key(box_min, np.int32), content_key(box_size, np.int32),
            DeviceTree.MAX_BRICK_TABLE)
    if any_shade:
        for key in reversed(_TREE_CACHE):
            if key[0] == tkey:
                _TREE_CACHE.move_to_end(key)
                _STATS["hits"] += 1
                return _TREE_CACHE[key]
        if shade is None:
            return None
    tree = _lru_get(_TREE_CACHE, (tkey, shade.key), TREE_CAPACITY,
                    lambda: DeviceTree(codes, flut_idx, root, left, right, box_min, box_size,
                                       shade))
    tree.shade = shade
    return tree


def _trace_shading(rows: int):
    """Trace-only shading: zero density, 1-channel degree-0 table."""
    return shading_for(np.zeros((rows, 2)), np.zeros(rows, np.int32), np.eye(3)[None], 0, 1)


def _in_range_or_zero(a, lo: float, hi: float) -> bool:
    """Every element 0 or of magnitude in [lo, hi] (numpy or torch)."""
    if isinstance(a, torch.Tensor):
        m = a.abs()
        return bool(((a == 0) | ((m >= lo) & (m <= hi))).all().item())
    m = np.abs(a)
    return bool(np.all((a == 0) | ((m >= lo) & (m <= hi))))


def fast_div_ok(og, dg) -> bool:
    """The operand ranges under which the cell walk's reciprocal-corrected
    division is exact for every crossing (artemis_rays.fast_div, bricks.cuh):
    grid-space origins 0 or in [2^-300, 2^300], directions 0 or in
    [2^-600, 2^300]. Real rays always qualify; anything else takes __ddiv_rn."""
    return _in_range_or_zero(og, 2.0 ** -300, 2.0 ** 300) and \
        _in_range_or_zero(dg, 2.0 ** -600, 2.0 ** 300)


class DeviceRays:
    def __init__(self, origins_g, dirs_g, dirs_w, t_min, t_max):
        og = np.asarray(origins_g, dtype=np.float64).reshape(-1, 3)
        dg = np.asarray(dirs_g, dtype=np.float64).reshape(-1, 3)
        self.og = upload(og, np.float64)
        self.dg = upload(dg, np.float64)
        self.dw = upload(np.asarray(dirs_w).reshape(-1, 3), np.float64) if dirs_w is not None \
            else self.dg
        self.n = self.og.shape[0]
        self.view = _lib.Rays(ptr(self.og), ptr(self.dg), ptr(self.dw), self.n, float(t_min),
                              float(t_max), int(fast_div_ok(og, dg)))

    @staticmethod
    def from_tensors(og, dg, dw, t_min=0.0, t_max=np.inf):
        r = DeviceRays.__new__(DeviceRays)
        r.og, r.dg, r.dw = og, dg, dw
        r.n = og.shape[0]
        r.view = _lib.Rays(ptr(og), ptr(dg), ptr(dw), r.n, float(t_min), float(t_max),
                           int(fast_div_ok(og, dg)) if r.n else 0)
        return r


def render_device(tree: DeviceTree, shade: DeviceShading, rays: DeviceRays, lambda_th,
                  sigma_dep, early_stop):
    """Device tensors (F fp32 (R,C), alpha fp64, depth fp64)."""
    L = _lib.lib()
    C_ = shade.view.channels
    F = empty((rays.n, C_), np.float32)
    A = empty(rays.n, np.float64)
    D = empty(rays.n, np.float64)
    if rays.n:
        check(L.artemis_render_rays(C.byref(tree.view), C.byref(shade.view), C.byref(rays.view),
                                    float(lambda_th), float(sigma_dep), int(bool(early_stop)),
                                    ptr(F), ptr(A), ptr(D), stream_handle()), "render_rays")
    return F, A, D


def render_rays(codes, flut_idx, root, left, right, box_min, box_size, origins_g, dirs_g,
                dirs_w, t_min, t_max, flut, rot_index, rot_inv, degree, channels, lambda_th,
                sigma_dep, early_stop, nthreads=1):
    shade = shading_for(flut, rot_index, rot_inv, degree, channels)
    tree = tree_for(codes, flut_idx, root, left, right, box_min, box_size, shade)
    rays = DeviceRays(origins_g, dirs_g, dirs_w, t_min, t_max)
    F, A, D = render_device(tree, shade, rays, lambda_th, sigma_dep, early_stop)
    return download(F).astype(np.float64), download(A), download(D)


def count_hits_device(tree: DeviceTree, rays: DeviceRays) -> torch.Tensor:
    L = _lib.lib()
    counts = empty(rays.n, np.int64)
    if rays.n:
        check(L.artemis_count_hits(C.byref(tree.view), C.byref(rays.view), ptr(counts),
                                   stream_handle()), "count_hits")
    return counts


def forward_fit_device(tree: DeviceTree, shade: DeviceShading, rays: DeviceRays):
    """(F, alpha, offsets (host int64), hit_idx, hit_t0, hit_t1) device tensors."""
    L = _lib.lib()
    counts = download(count_hits_device(tree, rays))
    offsets = np.zeros(rays.n + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    total = int(offsets[-1])
    d_off = upload(offsets, np.int64)
    hit_idx = empty(max(total, 1), np.int64)
    hit_t0 = empty(max(total, 1), np.float64)
    hit_t1 = empty(max(total, 1), np.float64)
    F = empty((rays.n, shade.view.channels), np.float32)
    A = empty(rays.n, np.float64)
    if rays.n:
        check(L.artemis_forward_fit(C.byref(tree.view), C.byref(shade.view), C.byref(rays.view),
                                    ptr(d_off), ptr(hit_idx), ptr(hit_t0), ptr(hit_t1), ptr(F),
                                    ptr(A), stream_handle()), "forward_fit")
    return F, A, offsets, hit_idx[:total], hit_t0[:total], hit_t1[:total]


def forward_fit(codes, flut_idx, root, left, right, box_min, box_size, origins_g, dirs_g,
                dirs_w, t_min, t_max, flut, rot_index, rot_inv, degree, channels, nthreads=1):
    shade = shading_for(flut, rot_index, rot_inv, degree, channels)
    tree = tree_for(codes, flut_idx, root, left, right, box_min, box_size, shade)
    rays = DeviceRays(origins_g, dirs_g, dirs_w, t_min, t_max)
    F, A, off, hi, h0, h1 = forward_fit_device(tree, shade, rays)
    return (download(F).astype(np.float64), download(A), off, download(hi), download(h0),
            download(h1))


def traverse_ray(codes, flut_idx, root, left, right, box_min, box_size, origin_g, dir_g,
                 t_min, t_max):
    fi = np.asarray(flut_idx)
    rows = int(fi.max()) + 1 if fi.size else 1
    # trace-only: zero density and a 1-channel degree-0 table (no shading work)
    tree = tree_for(codes, flut_idx, root, left, right, box_min, box_size, None, any_shade=True)
    if tree is not None:  # a cached tree of these arrays: its shading serves the trace
        shade = tree.shade
    else:
        shade = _trace_shading(rows)
        tree = tree_for(codes, flut_idx, root, left, right, box_min, box_size, shade)
    rays = DeviceRays(np.asarray(origin_g).reshape(1, 3), np.asarray(dir_g).reshape(1, 3), None,
                      t_min, t_max)
    _, _, _, hi, h0, h1 = forward_fit_device(tree, shade, rays)
    return download(hi), download(h0), download(h1)


def camera_rays_device(R, origin, fx, fy, cx, cy, width, height, lo, cell):
    """Exact device rays_for_camera + _grid_rays: (og, dg, dw) (W*H, 3) fp64."""
    L = _lib.lib()
    cam = camera_struct(R, origin, fx, fy, cx, cy, width, height, lo, cell)
    n = width * height
    og = empty((n, 3), np.float64)
    dg = empty((n, 3), np.float64)
    dw = empty((n, 3), np.float64)
    check(L.artemis_camera_rays(C.byref(cam), ptr(og), ptr(dg), ptr(dw), stream_handle()),
          "camera_rays")
    return og, dg, dw


def camera_struct(R, origin, fx, fy, cx, cy, width, height, lo, cell) -> _lib.Camera:
    cam = _lib.Camera()
    cam.R[:] = [float(v) for v in np.asarray(R, dtype=np.float64).reshape(9)]
    cam.origin[:] = [float(v) for v in np.asarray(origin, dtype=np.float64)]
    cam.fx, cam.fy, cam.cx, cam.cy = float(fx), float(fy), float(cx), float(cy)
    cam.width, cam.height = int(width), int(height)
    cam.lo[:] = [float(v) for v in np.asarray(lo, dtype=np.float64)]
    cam.cell[:] = [float(v) for v in np.asarray(cell, dtype=np.float64)]
    return cam


def backward_rays_device(offsets, hit_idx, hit_t0, hit_t1, dirs_w, rot_index, rot_inv, flut,
                         dldf, dlda, degree, channels, deterministic=True):
    """Device tensors in, device grad (n_flut, width) out; real type of flut."""
    L = _lib.lib()
    n_flut, width = int(flut.shape[0]), int(flut.shape[1])
    n_rays = int(offsets.numel()) - 1
    n_hits = int(hit_idx.numel())
    grad = torch.empty_like(flut)
    ws = workspace(L.artemis_backward_workspace_bytes(n_hits, n_flut))
    check(L.artemis_backward_rays(ptr(offsets), n_rays, ptr(hit_idx), ptr(hit_t0), ptr(hit_t1),
                                  n_hits, ptr(dirs_w), ptr(rot_index), ptr(rot_inv), ptr(flut),
                                  n_flut, width, ptr(dldf), ptr(dlda), flut.element_size(),
                                  int(degree), int(channels), int(bool(deterministic)),
                                  ptr(grad), ptr(ws), ws.numel(), stream_handle()),
          "backward_rays")
    return grad


def backward_rays(offsets, hit_idx, hit_t0, hit_t1, dirs_w, rot_index, rot_inv, flut, dldf, dlda,
                  degree, channels, deterministic=True, nthreads=1):
    """_core.pyx:661-755: gradient of the batch loss w.r.t. every FLUT entry
    (float32 instantiation when flut is float32, else float64); dldf/dlda are
    taken in flut's real type, as the reference's fused real_t requires."""
    fl = np.asarray(flut)
    rdt = np.float32 if fl.dtype == np.float32 else np.float64
    if fl.ndim != 2:
        raise ValueError("flut must be (N, H*C+1)")
    h = (int(degree) + 1) ** 2
    if fl.shape[1] != h * int(channels) + 1:
        raise ValueError("flut width must be (degree+1)^2 * channels + 1")
    off = np.ascontiguousarray(offsets, dtype=np.int64).reshape(-1)
    hi = np.ascontiguousarray(hit_idx, dtype=np.int64).reshape(-1)
    if hi.size == 0 or off.size <= 1 or int(np.diff(off).max(initial=0)) == 0:
        return np.zeros(fl.shape, dtype=rdt)
    g = backward_rays_device(
        upload(off, np.int64), upload(hi, np.int64),
        upload(np.asarray(hit_t0).reshape(-1), np.float64),
        upload(np.asarray(hit_t1).reshape(-1), np.float64),
        upload(np.asarray(dirs_w).reshape(-1, 3), np.float64),
        upload(np.asarray(rot_index).reshape(-1), np.int32),
        upload(np.asarray(rot_inv).reshape(-1, 9), np.float64),
        upload(fl, rdt), upload(np.asarray(dldf).reshape(-1, int(channels)), rdt),
        upload(np.asarray(dlda).reshape(-1), rdt), degree, channels, deterministic)
    return download(g)
