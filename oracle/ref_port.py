"""CPU BASELINE (test/bench infrastructure only): the reference's per-frame
CPU path, for timing beside the GPU.

The reference's kernels run from its own compiled Cython module
(oracle/_ref/_core*.so, built from /root/reference by build_ref.sh). Its
numpy stages -- warp_voxels (animvox/rigging.py:327-397),
resolve_collisions (:419-459), build_octree's orchestration
(animvox/volume.py:240-250) and rays_for_camera (animvox/geometry.py:242-263)
-- cannot travel to the GPU box with the read-only reference tree, so they
are restated here with the same numpy calls and the same per-group Python
loops, which is where the reference spends its warp/resolve time
(SURVEY.md section 6.3). bench.py --impl reference and the cpu_baseline leg
use this module; the product never imports it.
"""

from __future__ import annotations

import glob
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def load_reference_core():
    """The reference's compiled kernels module, or None if not built."""
    ref = os.path.join(HERE, "_ref")
    if not glob.glob(os.path.join(ref, "_core*.so")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import _core  # noqa: E402

    return _core


class RefFrame:
    """One posed frame through the reference CPU path, stage-timed."""

    def __init__(self, scene, core=None, nthreads=None):
        self.sc = scene
        self.core = core or load_reference_core()
        if self.core is None:
            import oracle

            self.core = oracle
            self.kind = "port"
        else:
            self.kind = "reference"
        self.nthreads = nthreads or os.cpu_count() or 1
        self.flut = scene.flut64()
        self.sigma = np.ascontiguousarray(self.flut[:, -1])

    # rigging.warp_voxels numerics and collision groups
    def warp(self, delta_mats):
        sc = self.sc
        cell = (sc.hi - sc.lo) / sc.resolution
        centers = sc.lo + (sc.cells.astype(np.float64) + 0.5) * cell
        n = centers.shape[0]
        pos = np.zeros((n, 3))
        jidx, w = sc.skin_idx, sc.skin_w
        for k in range(jidx.shape[1]):
            on = jidx[:, k] >= 0
            if not on.any():
                continue
            blk = delta_mats[jidx[on, k]]
            moved = np.einsum("nij,nj->ni", blk[:, :3, :3], centers[on]) + blk[:, :3, 3]
            pos[on] += w[on, k, None] * moved
        best = np.argmax(w, axis=1)
        rj = jidx[np.arange(n), best].astype(np.int32)
        rj[rj < 0] = 0
        g = np.floor((pos - sc.lo) / cell).astype(np.int64)
        inside = np.all((g >= 0) & (g < sc.resolution), axis=1)
        g[~inside] = -1
        groups = []
        ib = np.flatnonzero(inside)
        if ib.size:
            codes = self.core.morton_encode(g[ib])
            order = np.argsort(codes, kind="stable")
            sc_ = codes[order]
            cut = np.flatnonzero(sc_[1:] != sc_[:-1]) + 1
            for a, b in zip(np.concatenate([[0], cut]), np.concatenate([cut, [sc_.size]])):
                if b - a >= 2:
                    groups.append(ib[order[a:b]])
        return pos, g.astype(np.int32), inside, rj, groups

    # rigging.resolve_collisions
    def resolve(self, cells, inside):
        ib = np.flatnonzero(inside)
        codes = self.core.morton_encode(cells[ib])
        sig = self.sigma[ib]
        order = np.lexsort((ib, -sig, codes))
        sc_ = codes[order]
        canon = ib[order]
        cut = np.flatnonzero(sc_[1:] != sc_[:-1]) + 1
        starts = np.concatenate([[0], cut])
        ends = np.concatenate([cut, [sc_.size]])
        winners = canon[starts]
        rows = []
        for a, b in zip(starts, ends):
            if b - a >= 2:
                blk = np.empty((b - a - 1, 2), dtype=np.int64)
                blk[:, 0] = canon[a]
                blk[:, 1] = canon[a + 1:b]
                rows.append(blk)
        pairs = np.concatenate(rows) if rows else np.empty((0, 2), np.int64)
        return cells[winners].astype(np.int32), winners.astype(np.int64), pairs

    # volume.build_octree orchestration over the reference kernels
    def build(self, cells, flut_indices):
        codes = self.core.morton_encode(cells.astype(np.int64))
        order = self.core.sort_order(codes, nthreads=self.nthreads)
        codes = np.ascontiguousarray(codes[order])
        fi = np.ascontiguousarray(flut_indices.astype(np.uint32)[order])
        if np.any(codes[1:] == codes[:-1]):
            raise RuntimeError("duplicate Morton code")
        root, left, right, bmin, bsize = self.core.build_tree(codes, nthreads=self.nthreads)
        return codes, fi, int(root), left, right, bmin, bsize

    # geometry.rays_for_camera + render._grid_rays
    def rays(self, cam, rows=None):
        R, origin = cam.cam_to_world()
        u = np.arange(cam.width) + 0.5
        v = np.arange(cam.height) + 0.5
        if rows is not None:
            v = v[rows]
        uu, vv = np.meshgrid(u, v)
        d = np.stack([(uu - cam.cx) / cam.fx, (vv - cam.cy) / cam.fy, np.ones_like(uu)],
                     axis=-1).reshape(-1, 3)
        d = d @ R.T
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        o = np.broadcast_to(origin, d.shape)
        cell = (self.sc.hi - self.sc.lo) / self.sc.resolution
        return (np.ascontiguousarray((o - self.sc.lo) / cell), np.ascontiguousarray(d / cell),
                np.ascontiguousarray(d))

    def frame(self, tables, cams, row_stride: int = 1):
        """Stage seconds for one posed frame: warp + rebuild once, then every
        camera in `cams` (one camera, or a frame's views / stereo eyes)
        rendered in full (row_stride > 1 renders every row_stride-th row
        and scales the render time; the bench does not use it)."""
        if not isinstance(cams, (list, tuple)):
            cams = [cams]
        t = {}
        t0 = time.perf_counter()
        pos, cells, inside, rj, groups = self.warp(tables.delta_mats)
        t1 = time.perf_counter()
        live, win, pairs = self.resolve(cells, inside)
        tree = self.build(live, win)
        t2 = time.perf_counter()
        render = 0.0
        rays = 0
        for cam in cams:
            t3 = time.perf_counter()
            rows = np.arange(0, cam.height, row_stride)
            og, dg, dw = self.rays(cam, rows)
            self.core.render_rays(*tree, og, dg, dw, 0.0, np.inf, self.flut, rj,
                                  tables.rot_inv, self.sc.degree, self.sc.channels,
                                  self.sc.lambda_th, self.sc.sigma_dep, True, self.nthreads)
            render += (time.perf_counter() - t3) * cam.height / rows.size
            rays += int(og.shape[0])
        t["warp"] = t1 - t0
        t["build-octree"] = t2 - t1
        t["volume-render"] = render
        t["rays_sampled"] = rays
        return t
