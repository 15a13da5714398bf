"""Make the reference package (`animvox`) run its hot path on the B200.

The reference binds its kernel backend and its hot-path functions BY NAME at
import time (animvox/backend.py:19-31; `from .backend import kernels` in
volume.py:17, render.py:19, fit.py:22; `from .rigging import warp_voxels,
resolve_collisions` and `from .volume import build_octree` in render.py:22-31,
fit.py:25-34; `from .render import timed_render_frame` in cli.py:22 and
service.py:37). `install()` rebinds every one of those names, without
editing the reference, to:

  kernels                              -> paper_2202_05628_b200.kernels
  rigging.warp_voxels                  -> pipeline.warp_voxels
  rigging.resolve_collisions           -> pipeline.resolve_collisions
  volume.build_octree                  -> pipeline.build_octree
  render.posed_octree / render_view /
  render_frame / timed_render_frame    -> pipeline.* (device rays, device tree)

and makes the drop-ins return the reference's own result classes and raise
its own exception classes. `uninstall()` restores the original bindings.

  assetio.load_asset / load_asset_file -> assetio.* (native rig decode,
                                          device-resident leaves + FLUT)

`kernels.backward_rays` is the B200 gradient kernel, so fit.py's training
loop (forward_fit + backward_rays per batch) runs on the device too.
"""

from __future__ import annotations

import importlib
import sys

from . import assetio as _assetio
from . import kernels as _kernels
from . import pipeline as _pipeline
from . import types as _types

_SAVED: dict = {}

# (module, attribute, replacement) rebinding table
_TARGETS = (
    ("backend", "kernels", _kernels),
    ("volume", "kernels", _kernels),
    ("render", "kernels", _kernels),
    ("fit", "kernels", _kernels),
    ("rigging", "warp_voxels", _pipeline.warp_voxels),
    ("rigging", "resolve_collisions", _pipeline.resolve_collisions),
    ("render", "warp_voxels", _pipeline.warp_voxels),
    ("render", "resolve_collisions", _pipeline.resolve_collisions),
    ("fit", "warp_voxels", _pipeline.warp_voxels),
    ("fit", "resolve_collisions", _pipeline.resolve_collisions),
    ("volume", "build_octree", _pipeline.build_octree),
    ("render", "build_octree", _pipeline.build_octree),
    ("fit", "build_octree", _pipeline.build_octree),
    ("render", "posed_octree", _pipeline.posed_octree),
    ("render", "render_view", _pipeline.render_view),
    ("render", "render_frame", _pipeline.render_frame),
    ("render", "timed_render_frame", _pipeline.timed_render_frame),
    ("fit", "render_view", _pipeline.render_view),
    ("cli", "timed_render_frame", _pipeline.timed_render_frame),
    ("service", "timed_render_frame", _pipeline.timed_render_frame),
    ("assetio", "load_asset", _assetio.load_asset),
    ("assetio", "load_asset_file", _assetio.load_asset_file),
    ("service", "load_asset", _assetio.load_asset),
)


def _module(pkg: str, name: str):
    full = f"{pkg}.{name}"
    if full in sys.modules:
        return sys.modules[full]
    try:
        return importlib.import_module(full)
    except ImportError:  # optional modules (service needs websockets)
        return None


def install(package: str = "animvox") -> list:
    """Rebind the reference's hot path to the B200 implementation; returns
    the list of (module, attribute) pairs that were rebound."""
    done = []
    for mod_name, attr, repl in _TARGETS:
        mod = _module(package, mod_name)
        if mod is None or not hasattr(mod, attr):
            continue
        key = (package, mod_name, attr)
        if key not in _SAVED:
            _SAVED[key] = getattr(mod, attr)
        setattr(mod, attr, repl)
        done.append((mod_name, attr))
    volume = _module(package, "volume")
    rigging = _module(package, "rigging")
    render = _module(package, "render")
    errors = _module(package, "errors")
    _SAVED.setdefault((package, "_factories"), dict(_types.FACTORIES))
    if volume is not None:
        _types.FACTORIES["VoxelOctree"] = volume.VoxelOctree
    if rigging is not None:
        _types.FACTORIES["WarpResult"] = rigging.WarpResult
        _types.FACTORIES["CollisionResolution"] = rigging.CollisionResolution
    if render is not None:
        _types.FACTORIES["FrameBuffers"] = render.FrameBuffers
        _types.FACTORIES["CharacterAsset"] = render.CharacterAsset
    geometry = _module(package, "geometry")
    if volume is not None:
        for n in ("Bounds", "VoxelSet", "FLUT"):
            _types.FACTORIES[n] = getattr(volume, n)
    if rigging is not None:
        for n in ("Skeleton", "SkinWeights"):
            _types.FACTORIES[n] = getattr(rigging, n)
    if geometry is not None:
        _types.FACTORIES["RigidTransform"] = geometry.RigidTransform
    if errors is not None:
        _SAVED.setdefault((package, "_errors"), {n: getattr(_pipeline, n) for n in
                                                  ("ContractViolation", "DuplicateMortonError",
                                                   "EmptyWarpError")})
        for n in ("ContractViolation", "DuplicateMortonError", "EmptyWarpError"):
            setattr(_pipeline, n, getattr(errors, n))
        _SAVED.setdefault((package, "_asset_errors"), dict(_assetio.ERRORS))
        for n in _assetio.ERRORS:
            _assetio.ERRORS[n] = getattr(errors, n)
    return done


def uninstall(package: str = "animvox") -> None:
    for key, orig in list(_SAVED.items()):
        if len(key) != 3 or key[0] != package:
            continue
        pkg, mod_name, attr = key
        mod = _module(pkg, mod_name)
        if mod is not None:
            setattr(mod, attr, orig)
        del _SAVED[(pkg, mod_name, attr)]
    fac = _SAVED.pop((package, "_factories"), None)
    if fac is not None:
        _types.FACTORIES.clear()
        _types.FACTORIES.update(fac)
    aerrs = _SAVED.pop((package, "_asset_errors"), None)
    if aerrs is not None:
        _assetio.ERRORS.update(aerrs)
    errs = _SAVED.pop((package, "_errors"), None)
    if errs is not None:
        for n, cls in errs.items():
            setattr(_pipeline, n, cls)
