"""Device-resident character ingestion.

The reference loads a .nvo container (animvox/assetio.py:86-136) on the
host: Morton decode + scatter of the leaf table, an f32 -> f64 copy of the
FLUT block, and a per-voxel Python loop over the rig block
(assetio.py:158-202, seconds at ~1M voxels). Here:

* the header and extents are validated natively (artemis_asset_probe);
* the leaf table and the f32 FLUT block are copied to the device exactly as
  they lie in the file (one pinned staging buffer, one H2D), the leaves
  decoded and scattered to their FLUT rows on the device with the
  permutation check (artemis_asset_decode_leaves), the FLUT split into the
  render layout (artemis_flut_split_f32);
* the rig block is decoded natively in one pass (artemis_asset_decode_rig).

`load_device(data)` returns a DeviceAsset whose FramePipeline is built from
those device buffers (no second upload). `load_asset(data)` /
`load_asset_file(path)` are drop-ins for the reference's loaders: they
return the reference's CharacterAsset (bit-identical arrays, the reference's
exception classes in its validation order) and register the already
device-resident pipeline for that asset, so the first render_frame /
timed_render_frame on it (CLI `animate`/`bench`, the service) renders
straight away.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from . import kinematics as KM
from . import types as T
from ._lib import check
from .device import empty, ptr, stream_handle
from .errors import (AssetFormatError, ContractViolation, CountMismatchError,
                     MagicMismatchError, TruncatedAssetError)

# exception classes by reference name (install.py swaps in the reference's)
ERRORS = {
    "AssetFormatError": AssetFormatError,
    "TruncatedAssetError": TruncatedAssetError,
    "MagicMismatchError": MagicMismatchError,
    "CountMismatchError": CountMismatchError,
}

_STATUS = {
    _lib.ASSET_TRUNC_HEADER: ("TruncatedAssetError", "file ends inside header"),
    _lib.ASSET_BAD_MAGIC: ("MagicMismatchError", "magic != b'NVO1'"),
    _lib.ASSET_BAD_VERSION: ("AssetFormatError", "unsupported container version"),
    _lib.ASSET_ZERO_COUNT: ("CountMismatchError", "declared voxel count is zero"),
    _lib.ASSET_TRUNC_LEAVES: ("TruncatedAssetError", "file ends inside leaf table"),
    _lib.ASSET_TRUNC_FLUT: ("TruncatedAssetError", "file ends inside FLUT block"),
    _lib.ASSET_RIG_OFFSET: ("CountMismatchError", "rig offset does not follow the FLUT block"),
    _lib.ASSET_TRUNC_RIG: ("TruncatedAssetError", "file ends inside rig block"),
    _lib.ASSET_TRAILING: ("CountMismatchError", "trailing bytes after the asset"),
}


def _raise_status(status: int) -> None:
    if status == _lib.OK:
        return
    if status in _STATUS:
        name, msg = _STATUS[status]
        raise ERRORS[name](msg)
    check(status, "asset")


def _as_bytes(data) -> np.ndarray:
    if isinstance(data, (str, os.PathLike)):
        with open(data, "rb") as fh:
            data = fh.read()
    return np.frombuffer(data, dtype=np.uint8)


class DeviceAsset:
    """A .nvo character resident on the device, plus its host-side rig."""

    def __init__(self, info, cells, coef, sigma, names, parents, bind, joint_idx, weights):
        self.info = info
        self.resolution = int(info.resolution)
        self.count = int(info.count)
        self.degree, self.channels = int(info.degree), int(info.channels)
        self.lo = np.array(info.lo[:], dtype=np.float64)
        self.hi = np.array(info.hi[:], dtype=np.float64)
        self.cells, self.coef, self.sigma = cells, coef, sigma
        self.names, self.parents, self.bind = names, parents, bind
        self.joint_idx, self.weights = joint_idx, weights

    @property
    def rigged(self) -> bool:
        return self.parents is not None

    def rig(self) -> KM.Rig | None:
        if not self.rigged:
            return None
        return KM.Rig(parents=self.parents, bind_q=self.bind[:, :4].copy(),
                      bind_t=self.bind[:, 4:].copy())

    def pipeline(self):
        """FramePipeline over the device-resident buffers (no re-upload)."""
        from .frame import FramePipeline

        if self.rigged:
            jidx, w = self.joint_idx, self.weights
        else:
            jidx = np.zeros((self.count, 1), np.int32)
            w = np.ones((self.count, 1))
        return FramePipeline(self.cells, jidx, w, None, self.degree, self.channels,
                             self.resolution, self.lo, self.hi, rig=self.rig(),
                             device_flut=(self.coef, self.sigma))


def load_device(data) -> DeviceAsset:
    """Parse a .nvo container (bytes or path) into device memory."""
    buf = _as_bytes(data)
    L = _lib.load_library()
    info = _lib.AssetInfo()
    _raise_status(L.artemis_asset_probe(buf.ctypes.data, buf.size, C.byref(info)))
    L = _lib.lib()
    n, width = int(info.count), int(info.width)
    lo_b, hi_b = int(info.leaf_offset), int(info.flut_end)
    # leaf table + FLUT block: one pinned staging copy, one H2D
    stage = torch.empty(hi_b - lo_b, dtype=torch.uint8, pin_memory=True)
    stage.numpy()[:] = buf[lo_b:hi_b]
    blob = stage.to("cuda", non_blocking=True)
    st = stream_handle()
    cells = empty((n, 3), np.int32)
    seen = torch.empty(4 * n, dtype=torch.uint8, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    check(L.artemis_asset_decode_leaves(ptr(blob), n, ptr(cells), ptr(seen), seen.numel(),
                                        ptr(bad), st), "asset leaves")
    coef = empty((n, max(width - 1, 1)), np.float32)
    sigma = empty(n, np.float64)
    flut_dev = blob[int(info.flut_offset) - lo_b:]
    check(L.artemis_flut_split_f32(ptr(flut_dev), n, width, ptr(coef), ptr(sigma), st),
          "flut_split")
    if int(bad.item()):
        raise ERRORS["CountMismatchError"]("leaf table indices are not a permutation")
    rig = _lib.AssetRig()
    _raise_status(L.artemis_asset_decode_rig(buf.ctypes.data, buf.size, C.byref(info),
                                             C.byref(rig), None, None, None, None, None, None))
    names = parents = bind = jidx = w = None
    if int(info.rig_offset):
        J, K = int(rig.n_joints), int(rig.k_max)
        parents = np.empty(J, np.int32)
        bind = np.empty((J, 7), np.float64)
        raw = np.empty(max(int(rig.name_bytes), 1), np.uint8)
        offs = np.empty(J + 1, np.int32)
        jidx = np.empty((n, K), np.int32)
        w = np.empty((n, K), np.float64)
        _raise_status(L.artemis_asset_decode_rig(buf.ctypes.data, buf.size, C.byref(info),
                                                 C.byref(rig), parents.ctypes.data,
                                                 bind.ctypes.data, raw.ctypes.data,
                                                 offs.ctypes.data, jidx.ctypes.data,
                                                 w.ctypes.data))
        rb = raw.tobytes()
        names = tuple(rb[offs[j]:offs[j + 1]].decode("utf-8") for j in range(J))
    torch.cuda.current_stream().synchronize()
    del blob, seen
    return DeviceAsset(info, cells, coef, sigma, names, parents, bind, jidx, w)


def load_asset(data):
    """Drop-in for animvox.assetio.load_asset (assetio.py:86-136)."""
    buf = _as_bytes(data)
    da = load_device(buf)
    info, n, width = da.info, da.count, int(da.info.width)
    flut = np.frombuffer(buf, dtype="<f4", count=n * width,
                         offset=int(info.flut_offset)).reshape(n, width).astype(np.float64)
    bounds = T.make("Bounds", lo=da.lo.copy(), hi=da.hi.copy())
    voxels = T.make("VoxelSet", resolution=da.resolution, bounds=bounds,
                    cells=da.cells.cpu().numpy())
    fl = T.make("FLUT", data=flut, degree=da.degree, channels=da.channels)
    skeleton = weights = None
    if da.rigged:
        binds = tuple(T.make("RigidTransform", rotation=np.array(b[:4]), translation=np.array(b[4:]))
                      for b in da.bind)
        skeleton = T.make("Skeleton", names=da.names, parents=da.parents, bind_local=binds)
        weights = T.make("SkinWeights", joint_indices=da.joint_idx, weights=da.weights)
    asset = T.make("CharacterAsset", voxels=voxels, flut=fl, skeleton=skeleton, weights=weights)
    try:  # the character is already on the device: hand its pipeline to the renderers
        from . import pipeline as PL

        PL.DEVICE_ASSETS.adopt(asset, da.pipeline())
    except (ContractViolation, ValueError):
        pass
    return asset


def load_asset_file(path):
    """Drop-in for animvox.assetio.load_asset_file."""
    return load_asset(path)
