"""Device-resident frame pipeline (the throughput path).

One ``FramePipeline`` holds a character on the device -- canonical cells,
skin weights, the FLUT split into fp32 SH coefficients and fp64 density --
and renders posed frames with ``artemis_frame_run``: warp -> stable onesweep
sort -> collision resolve -> Karras build -> tile-ordered render with
in-kernel camera rays, all stream-ordered, the in-bounds / live counts
never leaving the device, and the whole sequence captured once as a CUDA
graph and replayed for every later pose/camera of the same image size.

Host work per frame is what the reference also does on the host: forward
kinematics over J joints (kinematics.pose_tables, rigging.py:228-247,
343-347) and the camera set-up.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from . import kernels as K
from . import kinematics as KM
from ._lib import check
from .device import download, empty, ptr, upload


class FramePipeline:
    def __init__(self, cells, skin_idx, skin_w, flut, degree: int, channels: int,
                 resolution: int, lo, hi, rig: KM.Rig | None = None, max_joints: int | None = None,
                 stream: torch.cuda.Stream | None = None, device_flut=None):
        """Host arrays are uploaded once; device tensors (cells int32 (N,3),
        skin idx int32 / weights fp64 (N,K)) and `device_flut` = (coef fp32
        (N, W-1), sigma fp64 (N)) are used in place (assetio.load_device)."""
        L = _lib.lib()
        self.stream = stream or torch.cuda.Stream()
        self.n = int(cells.shape[0])
        self.degree, self.channels = int(degree), int(channels)
        self.resolution = int(resolution)
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        self.cell = (self.hi - self.lo) / self.resolution
        self.rig = rig
        self._canon = KM.canonical_globals(rig) if rig is not None else None
        self._native_fk = None  # KM.NativePoseTables once checked against numpy

        def dev(a, dt):
            if isinstance(a, torch.Tensor):
                return a.contiguous()
            return upload(np.ascontiguousarray(a, dtype=dt), dt)

        with torch.cuda.stream(self.stream):
            self.d_cells = dev(cells, np.int32)
            self.d_jidx = dev(skin_idx, np.int32)
            self.d_w = dev(skin_w, np.float64)
            if device_flut is not None:
                self.coef, self.sigma = device_flut
            else:
                fl = np.asarray(flut)
                width = fl.shape[1]
                self.coef = empty((self.n, width - 1), np.float32)
                self.sigma = empty(self.n, np.float64)
                sh = self.stream.cuda_stream or None
                if fl.dtype == np.float32:
                    d_fl = upload(fl, np.float32)
                    check(L.artemis_flut_split_f32(ptr(d_fl), self.n, width, ptr(self.coef),
                                                   ptr(self.sigma), sh), "flut_split")
                else:
                    d_fl = upload(fl, np.float64)
                    check(L.artemis_flut_split_f64(ptr(d_fl), self.n, width, ptr(self.coef),
                                                   ptr(self.sigma), sh), "flut_split")
                self.stream.synchronize()
                del d_fl
        a = _lib.Asset()
        a.n_voxels = self.n
        a.resolution = self.resolution
        a.slots = int(self.d_jidx.shape[1])
        a.max_joints = int(max_joints or (rig.n_joints if rig is not None else 1))
        a.degree, a.channels = self.degree, self.channels
        a.lo[:] = [float(v) for v in self.lo]
        a.hi[:] = [float(v) for v in self.hi]
        a.cells, a.joint_idx, a.weights = ptr(self.d_cells), ptr(self.d_jidx), ptr(self.d_w)
        a.coef, a.sigma = ptr(self.coef), ptr(self.sigma)
        self._asset = a
        h = C.c_void_p()
        check(L.artemis_frame_create(C.byref(a), C.byref(h)), "frame_create")
        self._h = h
        self._outs = {}

    # -- construction helpers -------------------------------------------------
    @classmethod
    def from_scene(cls, scene, **kw) -> "FramePipeline":
        return cls(scene.cells, scene.skin_idx, scene.skin_w, scene.flut32, scene.degree,
                   scene.channels, scene.resolution, scene.lo, scene.hi, rig=scene.rig, **kw)

    @classmethod
    def from_asset(cls, asset, **kw) -> "FramePipeline":
        """From a reference CharacterAsset (render.py:106-126)."""
        v = asset.voxels
        rig = KM.Rig.from_any(asset.skeleton) if asset.skeleton is not None else None
        if asset.weights is not None:
            idx, w = asset.weights.joint_indices, asset.weights.weights
        else:
            idx = np.zeros((len(v.cells), 1), np.int32)
            w = np.ones((len(v.cells), 1))
        return cls(v.cells, idx, w, asset.flut.data, asset.flut.degree, asset.flut.channels,
                   v.resolution, v.bounds.lo, v.bounds.hi, rig=rig, **kw)

    # -- per frame --------------------------------------------------------------
    def tables(self, pose) -> KM.PoseTables:
        pose = KM.PoseSpec.from_any(pose)
        if self._native_fk is None:
            self._native_fk = (KM.NativePoseTables(self.rig, self._canon)
                               if KM.NativePoseTables.agrees() else False)
        if self._native_fk:
            return self._native_fk(pose)
        return KM.pose_tables(self.rig, pose, canonical=self._canon)

    def camera(self, cam) -> _lib.Camera:
        cam = KM.PinholeCamera.from_any(cam)
        R, origin = cam.cam_to_world()
        return K.camera_struct(R, origin, cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height,
                               self.lo, self.cell)

    def outputs(self, width: int, height: int, maps64: bool = False):
        key = (width, height, bool(maps64))
        if key not in self._outs:
            with torch.cuda.stream(self.stream):
                n = width * height
                mt = np.float64 if maps64 else np.float32
                self._outs[key] = (empty((n, self.channels), np.float32), empty(n, mt),
                                   empty(n, mt))
        return self._outs[key]

    def run(self, pose, camera, *, lambda_th: float = 1e-4, sigma_dep: float = 5.0,
            early_stop: bool = True, graph: bool = True, parity: bool = False, tables=None,
            out=None, tiles: tuple | None = None, maps64: bool = False,
            reuse_tree: bool = False):
        """Enqueue one frame on self.stream; returns device (F, alpha, depth)
        (row-major pixels; F fp32, alpha/depth fp32, or fp64 with exact
        entry distances when `maps64`). `pose` None renders the canonical
        cells. `tiles` = (start, stride) renders only that tile shard
        (parallel.py). `reuse_tree` renders another view of the tree the
        previous run built for the same pose (multi-view, stereo eyes)."""
        L = _lib.lib()
        cam = camera if isinstance(camera, _lib.Camera) else self.camera(camera)
        if tiles is not None:
            cam.tile_start, cam.tile_stride = int(tiles[0]), int(tiles[1])
        if pose is None or self.rig is None:
            aff = rot = None
            nj = 1
        else:
            t = tables if tables is not None else self.tables(pose)
            aff = np.ascontiguousarray(t.affine34)
            rot = np.ascontiguousarray(t.rot_inv.reshape(-1, 9))
            nj = int(aff.shape[0])
        F, A, D = out if out is not None else self.outputs(cam.width, cam.height, maps64)
        if (A.dtype == torch.float64) != bool(maps64):
            raise ValueError("alpha/depth buffers must be float64 exactly when maps64")
        flags = ((1 if early_stop else 0) | (2 if graph else 0) | (4 if parity else 0)
                 | (8 if maps64 else 0) | (16 if reuse_tree else 0))
        check(L.artemis_frame_run(self._h, aff.ctypes.data if aff is not None else None,
                                  rot.ctypes.data if rot is not None else None, nj, C.byref(cam),
                                  float(lambda_th), float(sigma_dep), flags, ptr(F), ptr(A),
                                  ptr(D), self.stream.cuda_stream or None), "frame_run")
        cur = torch.cuda.current_stream()
        if cur != self.stream:
            cur.wait_stream(self.stream)  # consumers on the caller's stream see the frame
        return F, A, D

    def host_frame64(self, F, A, D, width: int, height: int):
        """A maps64 frame on this pipeline's stream -> freshly allocated host
        arrays in the reference's FrameBuffers layout (render.py:359-363):
        features float64 (h, w, C), alpha and depth float64 (h, w). Only the
        covered pixels' bounding box of F crosses PCIe (pinned staging) and is
        widened to float64 natively on several host threads; the rest of the
        features array is zero (np.zeros pages, untouched)."""
        L = _lib.lib()
        C_ = self.channels
        n = width * height
        key = ("api64", width, height)
        if not hasattr(self, "_api_bufs"):
            self._api_bufs = {}
        if key not in self._api_bufs:
            with torch.cuda.stream(self.stream):
                dbox = torch.empty(4, dtype=torch.int32, device="cuda")
            self._api_bufs[key] = dict(
                dbox=dbox, box=torch.empty(4, dtype=torch.int32, pin_memory=True),
                F=torch.empty(n * C_, dtype=torch.float32, pin_memory=True),
                A=torch.empty(n, dtype=torch.float64, pin_memory=True),
                D=torch.empty(n, dtype=torch.float64, pin_memory=True))
        b = self._api_bufs[key]
        st = self.stream.cuda_stream or None
        check(L.artemis_frame_bbox(ptr(A), ptr(D), 1, width, height, ptr(b["dbox"]), st),
              "frame_bbox")
        with torch.cuda.stream(self.stream):
            b["box"].copy_(b["dbox"], non_blocking=True)
            b["A"].copy_(A.reshape(-1), non_blocking=True)
            b["D"].copy_(D.reshape(-1), non_blocking=True)
        self.stream.synchronize()
        x0, y0, x1, y1 = (int(v) for v in b["box"])
        features = np.zeros((height, width, C_), dtype=np.float64)
        if x1 >= 0:
            rows, cols = y1 - y0 + 1, (x1 - x0 + 1) * C_
            check(L.artemis_copy_rect_d2h(b["F"].data_ptr(), ptr(F), width * C_ * 4, x0 * C_ * 4,
                                          cols * 4, y0, rows, st), "copy_rect")
            self.stream.synchronize()
            off = (y0 * width + x0) * C_
            check(L.artemis_host_widen_f32(b["F"].data_ptr() + 4 * off, rows, cols, width * C_,
                                           features.ctypes.data + 8 * off, width * C_,
                                           max(1, min(16, os.cpu_count() or 1))), "widen")
        alpha = b["A"].numpy().reshape(height, width).copy()
        depth = b["D"].numpy().reshape(height, width).copy()
        return features, alpha, depth

    def view_outputs(self, width: int, height: int, n: int, maps64: bool = False):
        """Persistent per-view device outputs for run_views."""
        key = ("views", width, height, n, bool(maps64))
        if key not in self._outs:
            with torch.cuda.stream(self.stream):
                mt = np.float64 if maps64 else np.float32
                px = width * height
                self._outs[key] = [(empty((px, self.channels), np.float32), empty(px, mt),
                                    empty(px, mt)) for _ in range(n)]
        return self._outs[key]

    def run_views(self, pose, cameras, *, lambda_th: float = 1e-4, sigma_dep: float = 5.0,
                  early_stop: bool = True, graph: bool = True, tables=None,
                  maps64: bool = False, outs=None):
        """One pose, up to 8 views of one image size (configs[1] views,
        configs[4] stereo eyes): warp + rebuild once and ONE render launch
        whose ray queue interleaves the views' 8x4 tiles, so rays of
        different views over the same leaves share the FLUT rows in L2.
        Returns the views' device (F, alpha, depth) (persistent buffers,
        overwritten by the next call with the same shape)."""
        L = _lib.lib()
        cams = [c if isinstance(c, _lib.Camera) else self.camera(c) for c in cameras]
        n = len(cams)
        if not 1 <= n <= 8 or any((c.width, c.height) != (cams[0].width, cams[0].height)
                                  for c in cams):
            raise ValueError("run_views takes 1..8 cameras of one image size")
        if pose is None or self.rig is None:
            aff = rot = None
            nj = 1
        else:
            t = tables if tables is not None else self.tables(pose)
            aff = np.ascontiguousarray(t.affine34)
            rot = np.ascontiguousarray(t.rot_inv.reshape(-1, 9))
            nj = int(aff.shape[0])
        outs = outs if outs is not None else self.view_outputs(cams[0].width, cams[0].height, n,
                                                               maps64)
        carr = (_lib.Camera * n)(*cams)
        pa = (C.c_void_p * n)
        Fs, As, Ds = (pa(*[ptr(o[k]) for o in outs]) for k in range(3))
        flags = (1 if early_stop else 0) | (2 if graph else 0) | (8 if maps64 else 0)
        check(L.artemis_frame_run_views(self._h, aff.ctypes.data if aff is not None else None,
                                        rot.ctypes.data if rot is not None else None, nj,
                                        C.cast(carr, C.c_void_p), n, float(lambda_th),
                                        float(sigma_dep), flags, C.cast(Fs, C.c_void_p),
                                        C.cast(As, C.c_void_p), C.cast(Ds, C.c_void_p),
                                        self.stream.cuda_stream or None), "frame_run_views")
        cur = torch.cuda.current_stream()
        if cur != self.stream:
            cur.wait_stream(self.stream)
        return outs

    def render_views(self, pose, cameras, *, lambda_th: float = 1e-4, sigma_dep: float = 5.0,
                     early_stop: bool = True, graph: bool = True, tables=None):
        """One pose, several cameras (configs[1] views, configs[4] stereo
        eyes): warp + rebuild once, then the views rendered together
        (run_views; one render per camera when sizes differ or there are
        more than 8). Returns a list of device (F, alpha, depth) clones."""
        t = tables if tables is not None or pose is None or self.rig is None \
            else self.tables(pose)
        cams = [c if isinstance(c, _lib.Camera) else self.camera(c) for c in cameras]
        if 1 <= len(cams) <= 8 and all((c.width, c.height) == (cams[0].width, cams[0].height)
                                       for c in cams):
            res = self.run_views(pose, cams, lambda_th=lambda_th, sigma_dep=sigma_dep,
                                 early_stop=early_stop, graph=graph, tables=t)
            with torch.cuda.stream(self.stream):
                return [tuple(x.clone() for x in o) for o in res]
        outs = []
        for i, cam in enumerate(cams):
            F, A, D = self.run(pose, cam, lambda_th=lambda_th, sigma_dep=sigma_dep,
                               early_stop=early_stop, graph=graph, tables=t,
                               reuse_tree=i > 0)
            with torch.cuda.stream(self.stream):
                outs.append((F.clone(), A.clone(), D.clone()))
        return outs

    def run_stream(self, items, *, lambda_th: float = 1e-4, sigma_dep: float = 5.0,
                   early_stop: bool = True, readout: str = "box"):
        """Render a sequence of (pose, camera) frames to HOST memory.

        Yields (F, alpha, depth) host tensors (dense fp32 maps, row-major
        pixels), one triple per item, in order; a yielded triple stays valid
        until the generator is advanced. Frames are pipelined: frame k
        renders while frame k-1's result crosses PCIe on the copy engine.
        `readout` chooses what crosses PCIe (the maps are bit-identical):

        * "box" (default): the bounding box of the covered pixels (alpha > 0
          or finite depth; artemis_frame_bbox) united with the previous
          frame's box in the same host buffer, as three 2-D copies straight
          into persistent pinned dense maps (artemis_copy_rect_d2h): outside
          the union both frames are (0, 0, +inf). No host-side work.
        * "records": only the covered pixels, compacted on the device
          (artemis_frame_compact) and scattered into the dense maps on the
          host (artemis_host_expand) -- fewest bytes, host CPU work.
        * "dense": the whole maps, 4(C+2) bytes per pixel."""
        if readout == "dense":
            yield from self._run_stream_dense(items, lambda_th=lambda_th, sigma_dep=sigma_dep,
                                              early_stop=early_stop)
            return
        if readout == "box":
            yield from self._run_stream_box(items, lambda_th=lambda_th, sigma_dep=sigma_dep,
                                            early_stop=early_stop)
            return
        if readout != "records":
            raise ValueError("readout must be 'box', 'records' or 'dense'")
        L = _lib.lib()
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream()
            self._stream_bufs = {}
        cs = self._copy_stream
        C_ = self.channels
        R = C_ + 3
        threads = max(1, min(16, (os.cpu_count() or 2) // 2))
        self.last_stream_d2h_bytes = []

        def bufs(w, h, b):
            key = ("sparse", w, h, b)
            if key not in self._stream_bufs:
                n = w * h
                with torch.cuda.stream(self.stream):
                    dev = (empty((n, C_), np.float32), empty(n, np.float32), empty(n, np.float32))
                    drec = torch.empty(n * R, dtype=torch.int32, device="cuda")
                    dcnt = torch.zeros(1, dtype=torch.int64, device="cuda")
                    ws = torch.empty(L.artemis_compact_workspace_bytes(n), dtype=torch.uint8,
                                     device="cuda")
                hrec = torch.empty(n * R, dtype=torch.int32, pin_memory=True)
                hcnt = torch.zeros(1, dtype=torch.int64, pin_memory=True)
                dense = (torch.zeros((n, C_), dtype=torch.float32),
                         torch.zeros(n, dtype=torch.float32),
                         torch.full((n,), float("inf"), dtype=torch.float32))
                pix = [torch.empty(n, dtype=torch.int32), 0]  # dense buffer's covered pixels
                self._stream_bufs[key] = dict(dev=dev, drec=drec, dcnt=dcnt, ws=ws, hrec=hrec,
                                              hcnt=hcnt, dense=dense, pix=pix,
                                              counted=torch.cuda.Event(),
                                              copied=torch.cuda.Event(), n=0)
            return self._stream_bufs[key]

        def launch_copy(bb):  # frame's count is on the host: move exactly its records
            bb["counted"].synchronize()
            n = int(bb["hcnt"][0])
            bb["n"] = n
            cs.wait_event(bb["counted"])
            if n:
                with torch.cuda.stream(cs):
                    bb["hrec"][:n * R].copy_(bb["drec"][:n * R], non_blocking=True)
            bb["copied"].record(cs)
            self.last_stream_d2h_bytes.append(n * R * 4 + 8)

        def expand(bb):
            bb["copied"].synchronize()
            F, A, D = bb["dense"]
            pix = bb["pix"]
            n = bb["n"]
            check(L.artemis_host_expand(bb["hrec"].data_ptr() if n else None, n, C_,
                                        pix[0].data_ptr() if pix[1] else None, pix[1],
                                        F.data_ptr(), A.data_ptr(), D.data_ptr(),
                                        pix[0].data_ptr(), threads), "host_expand")
            pix[1] = n
            return bb["dense"]

        pending = []
        for k, (pose, camera) in enumerate(items):
            cam = camera if isinstance(camera, _lib.Camera) else self.camera(camera)
            bb = bufs(cam.width, cam.height, k % 2)
            self.stream.wait_event(bb["copied"])  # its records buffer has been read out
            F, A, D = self.run(pose, cam, lambda_th=lambda_th, sigma_dep=sigma_dep,
                               early_stop=early_stop, out=bb["dev"])
            n_pix = cam.width * cam.height
            check(L.artemis_frame_compact(ptr(F), ptr(A), ptr(D), 0, n_pix, C_, ptr(bb["drec"]),
                                          ptr(bb["dcnt"]), ptr(bb["ws"]), bb["ws"].numel(),
                                          self.stream.cuda_stream or None), "frame_compact")
            with torch.cuda.stream(self.stream):
                bb["hcnt"].copy_(bb["dcnt"], non_blocking=True)
            bb["counted"].record(self.stream)
            pending.append(bb)
            if len(pending) >= 2:
                launch_copy(pending[-2])
            if len(pending) >= 3:
                yield expand(pending.pop(0))
        if pending:  # the last frame's copy is not launched yet
            launch_copy(pending[-1])
        for bb in pending:
            yield expand(bb)

    def twin(self) -> "FramePipeline":
        """A second pipeline over the SAME device asset arrays (no upload) with
        its own frame state, stream and graphs: run_stream alternates frames
        between the two, so frame k+1's warp and rebuild start on the SMs
        frame k's render tail releases instead of after the whole render."""
        if getattr(self, "_twin", None) is None:
            self._twin = FramePipeline(self.d_cells, self.d_jidx, self.d_w, None, self.degree,
                                       self.channels, self.resolution, self.lo, self.hi,
                                       rig=self.rig, max_joints=int(self._asset.max_joints),
                                       device_flut=(self.coef, self.sigma))
        return self._twin

    def _run_stream_box(self, items, *, lambda_th, sigma_dep, early_stop):
        L = _lib.lib()
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream()
            self._stream_bufs = {}
        cs = self._copy_stream
        # frames alternate between this pipeline and its twin (buffer b is
        # always rendered by pipeline b) while the FLUT fits in half the L2:
        # then two frames in flight share it and frame k+1's rebuild fills
        # frame k's render tail (configs[0] stream 0.295 -> 0.209 ms/frame);
        # with a FLUT beyond L2 two renders in flight evict each other's rows
        # (configs[2] 1.54 -> 1.74 ms/frame), so one pipeline.
        # ARTEMIS_STREAM_TWIN=0/1 forces either.
        env = os.environ.get("ARTEMIS_STREAM_TWIN", "")
        l2 = getattr(torch.cuda.get_device_properties(self.coef.device), "L2_cache_size", 126 << 20)
        small = self.coef.numel() * self.coef.element_size() <= 0.5 * l2
        pipes = [self, self.twin()] if (env == "1" or (env != "0" and small)) else [self, self]
        C_ = self.channels
        self.last_stream_d2h_bytes = []

        def bufs(w, h, b):
            key = ("box", w, h, b)
            if key not in self._stream_bufs:
                n = w * h
                with torch.cuda.stream(self.stream):
                    dev = (empty((n, C_), np.float32), empty(n, np.float32), empty(n, np.float32))
                    dbox = torch.empty(4, dtype=torch.int32, device="cuda")
                hbox = torch.empty(4, dtype=torch.int32, pin_memory=True)
                dense = (torch.zeros((n, C_), dtype=torch.float32, pin_memory=True),
                         torch.zeros(n, dtype=torch.float32, pin_memory=True),
                         torch.full((n,), float("inf"), dtype=torch.float32, pin_memory=True))
                self._stream_bufs[key] = dict(dev=dev, dbox=dbox, hbox=hbox, dense=dense,
                                              prev=(1 << 30, 1 << 30, -1, -1), w=w, h=h,
                                              boxed=torch.cuda.Event(),
                                              copied=torch.cuda.Event())
            return self._stream_bufs[key]

        def launch_copy(bb):  # union of this frame's and the buffer's last box
            bb["boxed"].synchronize()
            x0, y0, x1, y1 = (int(v) for v in bb["hbox"])
            px0, py0, px1, py1 = bb["prev"]
            ux0, uy0, ux1, uy1 = min(x0, px0), min(y0, py0), max(x1, px1), max(y1, py1)
            bb["prev"] = (x0, y0, x1, y1)
            cs.wait_event(bb["boxed"])
            nbytes = 0
            if ux1 >= ux0 and uy1 >= uy0:
                w, rows = ux1 - ux0 + 1, uy1 - uy0 + 1
                st = cs.cuda_stream or None
                for dst, src, per in zip(bb["dense"], bb["dev"], (4 * C_, 4, 4)):
                    check(L.artemis_copy_rect_d2h(dst.data_ptr(), src.data_ptr(), bb["w"] * per,
                                                  ux0 * per, w * per, uy0, rows, st),
                          "copy_rect")
                nbytes = w * rows * 4 * (C_ + 2)
            bb["copied"].record(cs)
            self.last_stream_d2h_bytes.append(nbytes + 16)

        pending = []
        for k, (pose, camera) in enumerate(items):
            cam = camera if isinstance(camera, _lib.Camera) else self.camera(camera)
            bb = bufs(cam.width, cam.height, k % 2)
            pp = pipes[k % 2]
            pp.stream.wait_event(bb["copied"])  # its device maps have been read out
            F, A, D = pp.run(pose, cam, lambda_th=lambda_th, sigma_dep=sigma_dep,
                             early_stop=early_stop, out=bb["dev"])
            check(L.artemis_frame_bbox(ptr(A), ptr(D), 0, cam.width, cam.height, ptr(bb["dbox"]),
                                       pp.stream.cuda_stream or None), "frame_bbox")
            with torch.cuda.stream(pp.stream):
                bb["hbox"].copy_(bb["dbox"], non_blocking=True)
            bb["boxed"].record(pp.stream)
            pending.append(bb)
            if len(pending) >= 2:
                launch_copy(pending[-2])
            if len(pending) >= 3:
                out = pending.pop(0)
                out["copied"].synchronize()
                yield out["dense"]
        if pending:
            launch_copy(pending[-1])
        for bb in pending:
            bb["copied"].synchronize()
            yield bb["dense"]

    def _run_stream_dense(self, items, *, lambda_th, sigma_dep, early_stop, buffers: int = 2):
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream()
            self._stream_bufs = {}
        copy_stream = self._copy_stream
        pending = []
        for k, (pose, camera) in enumerate(items):
            cam = camera if isinstance(camera, _lib.Camera) else self.camera(camera)
            n = cam.width * cam.height
            b = k % buffers
            key = (cam.width, cam.height, b)
            if key not in self._stream_bufs:
                with torch.cuda.stream(self.stream):
                    d = (empty((n, self.channels), np.float32), empty(n, np.float32),
                         empty(n, np.float32))
                h = tuple(torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in d)
                self._stream_bufs[key] = (d, h, torch.cuda.Event(), torch.cuda.Event())
            dev_b, host_b, done_b, copied_b = self._stream_bufs[key]
            self.stream.wait_event(copied_b)  # device buffer b has been read out
            self.run(pose, cam, lambda_th=lambda_th, sigma_dep=sigma_dep,
                     early_stop=early_stop, out=dev_b)
            done_b.record(self.stream)
            copy_stream.wait_event(done_b)
            with torch.cuda.stream(copy_stream):
                for h, d in zip(host_b, dev_b):
                    h.copy_(d, non_blocking=True)
            copied_b.record(copy_stream)
            pending.append((host_b, copied_b))
            if len(pending) > 1:
                h, ev = pending.pop(0)
                ev.synchronize()
                yield h
        for h, ev in pending:
            ev.synchronize()
            yield h

    def counts(self):
        n_in, n_live = C.c_int64(), C.c_int64()
        check(_lib.lib().artemis_frame_counts(self._h, C.byref(n_in), C.byref(n_live),
                                              self.stream.cuda_stream or None), "frame_counts")
        return int(n_in.value), int(n_live.value)

    def profile(self, enable: bool = True) -> None:
        check(_lib.lib().artemis_frame_profile(self._h, int(bool(enable))), "frame_profile")

    def stage_ms(self) -> dict:
        """Per-stage device ms of the last eager profiled run."""
        ms = (C.c_float * 5)()
        check(_lib.lib().artemis_frame_stage_ms(self._h, ms), "frame_stage_ms")
        return dict(zip(("warp", "sort", "resolve", "build", "render"), [float(v) for v in ms]))

    def launches_per_frame(self) -> int:
        return int(_lib.lib().artemis_frame_launches(self._h))

    def tree(self):
        """Host copies of the last frame's tree (run with parity=True)."""
        ft = _lib.FrameTree()
        check(_lib.lib().artemis_frame_get_tree(self._h, C.byref(ft)), "frame_get_tree")
        n_in, n_live = self.counts()

        def grab(p, count, dtype, cols=1):
            a = np.empty((max(count, 0), cols), dtype=dtype)
            if count > 0:
                check(_lib.lib().artemis_copy_to_host(a.ctypes.data, p, a.nbytes,
                                                      self.stream.cuda_stream or None), "copy")
            return a if cols > 1 else a.reshape(-1)

        code_dt = np.uint32 if ft.code_bytes == 4 else np.uint64
        out = dict(
            n_in=n_in, n_live=n_live,
            codes=grab(ft.codes, n_live, code_dt).astype(np.uint64),
            flut_idx=grab(ft.flut_idx, n_live, np.uint32),
            left=grab(ft.left, n_live - 1, np.int32),
            right=grab(ft.right, n_live - 1, np.int32),
            box_min=grab(ft.box_min, n_live - 1, np.int32, 3),
            box_size=grab(ft.box_size, n_live - 1, np.int32, 3),
            rotation_joint=grab(ft.rotation_joint, self.n, np.int32),
        )
        out["root"] = 0 if n_live > 1 else ~0
        return out

    def set_output_peer(self, F=None, alpha=None, depth=None) -> None:
        """Tile-sharded frames write their pixels into these full-frame device
        tensors (the destination rank's, mapped over CUDA IPC / NVLink)
        instead of this pipeline's outputs; None restores the local ones.
        A sharded frame of another image size or map type is refused."""
        if F is None:
            check(_lib.lib().artemis_frame_set_output_peer(self._h, None, None, None, 0, 0),
                  "frame_set_output_peer")
            return
        n = int(alpha.numel())
        if F.numel() != n * self.channels or depth.numel() != n or depth.dtype != alpha.dtype:
            raise ValueError("peer maps must be (n, C) F and (n,) alpha/depth of one dtype")
        check(_lib.lib().artemis_frame_set_output_peer(
            self._h, ptr(F), ptr(alpha), ptr(depth), n, int(alpha.dtype == torch.float64)),
            "frame_set_output_peer")

    def set_tile_order(self, width: int, height: int, order) -> None:
        """Render the 8x4 ray tiles of a width x height image in `order` (a
        permutation of the row-major tile indices); the maps do not change."""
        o = np.ascontiguousarray(order, dtype=np.int32)
        check(_lib.lib().artemis_frame_set_tile_order(self._h, int(width), int(height),
                                                      o.ctypes.data), "frame_set_tile_order")

    def close(self):
        if getattr(self, "_twin", None) is not None:
            self._twin.close()
            self._twin = None
        if getattr(self, "_h", None):
            _lib.lib().artemis_frame_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ViewsReadout:
    """Dense pinned host copies of a fixed set of device frames (views of
    one size: multi-view / stereo / gathered tiles), refreshed per frame by
    the covered-pixel box of each view united with the box its host buffer
    last received (artemis_views_bbox + artemis_views_copy_union_d2h: two
    native calls per frame however many views). `mark(stream)` enqueues the
    boxes after the frame; `copy(copy_stream)` waits for them and issues the
    2-D copies; the host maps are valid once `copied` has completed."""

    def __init__(self, triples, width: int, height: int, channels: int, maps64: bool = False):
        L = _lib.lib()
        self.L = L
        self.n = len(triples)
        self.w, self.h, self.c = int(width), int(height), int(channels)
        self.maps64 = bool(maps64)
        mt = torch.float64 if maps64 else torch.float32
        n = self.w * self.h
        self.triples = list(triples)
        self.host = [(torch.zeros((n, self.c), dtype=torch.float32, pin_memory=True),
                      torch.zeros(n, dtype=mt, pin_memory=True),
                      torch.full((n,), float("inf"), dtype=mt, pin_memory=True))
                     for _ in range(self.n)]
        self.dbox = torch.empty((self.n, 4), dtype=torch.int32, device="cuda")
        self.hbox = torch.empty((self.n, 4), dtype=torch.int32, pin_memory=True)
        self.prev = np.tile(np.array([self.w, self.h, -1, -1], dtype=np.int32), (self.n, 1))
        pa = C.c_void_p * self.n
        self._A = pa(*[ptr(t[1]) for t in self.triples])
        self._D = pa(*[ptr(t[2]) for t in self.triples])
        p3 = C.c_void_p * (3 * self.n)
        self._dev = p3(*[ptr(x) for t in self.triples for x in t])
        self._host = p3(*[x.data_ptr() for t in self.host for x in t])
        self.boxed = None
        self.copied = None
        self.last_bytes = 0

    def mark(self, stream: torch.cuda.Stream) -> None:
        st = stream.cuda_stream or None
        check(self.L.artemis_views_bbox(C.cast(self._A, C.c_void_p), C.cast(self._D, C.c_void_p),
                                        self.n, int(self.maps64), self.w, self.h,
                                        ptr(self.dbox), st), "views_bbox")
        with torch.cuda.stream(stream):
            self.hbox.copy_(self.dbox, non_blocking=True)
        self.boxed = torch.cuda.Event()
        self.boxed.record(stream)

    def copy(self, copy_stream: torch.cuda.Stream) -> int:
        self.boxed.synchronize()
        copy_stream.wait_event(self.boxed)
        moved = C.c_int64(0)
        check(self.L.artemis_views_copy_union_d2h(
            self.n, self.hbox.data_ptr(), self.prev.ctypes.data, C.cast(self._dev, C.c_void_p),
            C.cast(self._host, C.c_void_p), self.w, self.h, self.c, int(self.maps64),
            C.byref(moved), copy_stream.cuda_stream or None), "views_copy")
        self.copied = torch.cuda.Event()
        self.copied.record(copy_stream)
        self.last_bytes = int(moved.value)
        return self.last_bytes
