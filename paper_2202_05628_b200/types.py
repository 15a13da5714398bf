"""Result types of the drop-in entry points.

Field names mirror the reference's dataclasses so callers (and the
reference's own code) can consume them unchanged:

* VoxelOctree          animvox/volume.py:186-209
* WarpResult           animvox/rigging.py:182-211
* CollisionResolution  animvox/rigging.py:214-221
* FrameBuffers         animvox/render.py:77-104
* RenderOptions        animvox/render.py:34-64
* VoxelSet, FLUT       animvox/volume.py:61-179 (what load_asset builds)
* RigidTransform       animvox/geometry.py (rotation quaternion, translation)
* Skeleton, SkinWeights  animvox/rigging.py:32-180
* CharacterAsset       animvox/render.py:106-126

When the reference package is installed into (install.py), the factories
below build the reference's own classes instead, so identity checks such
as ``isinstance(x, animvox.volume.VoxelOctree)`` keep passing.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ContractViolation


@dataclass(frozen=True)
class Bounds:
    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.lo, dtype=np.float64)
        hi = np.asarray(self.hi, dtype=np.float64)
        if lo.shape != (3,) or hi.shape != (3,) or not np.all(hi > lo):
            raise ContractViolation("bounds must be 3-vectors with positive extent")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    def cell_size(self, resolution: int) -> np.ndarray:
        return (self.hi - self.lo) / resolution


@dataclass(frozen=True)
class VoxelOctree:
    resolution: int
    bounds: object
    codes: np.ndarray
    flut_idx: np.ndarray
    root: int
    left: np.ndarray = field(repr=False)
    right: np.ndarray = field(repr=False)
    box_min: np.ndarray = field(repr=False)
    box_size: np.ndarray = field(repr=False)

    def __len__(self) -> int:
        return self.codes.shape[0]

    @property
    def cell_size(self) -> np.ndarray:
        return self.bounds.cell_size(self.resolution)


@dataclass(frozen=True)
class WarpResult:
    resolution: int
    bounds_lo: np.ndarray
    cell_size: np.ndarray
    positions: np.ndarray
    cells: np.ndarray
    rotations: np.ndarray
    rotation_joint: np.ndarray
    joint_rot_inv: np.ndarray
    in_bounds: np.ndarray
    collision_groups: tuple

    @property
    def n_voxels(self) -> int:
        return self.positions.shape[0]

    @property
    def dropped(self) -> int:
        return int(self.n_voxels - np.count_nonzero(self.in_bounds))


@dataclass(frozen=True)
class CollisionResolution:
    cells: np.ndarray
    flut_indices: np.ndarray
    pairs: np.ndarray


@dataclass(frozen=True)
class FrameBuffers:
    features: np.ndarray
    alpha: np.ndarray
    depth: np.ndarray

    @property
    def height(self) -> int:
        return self.alpha.shape[0]

    @property
    def width(self) -> int:
        return self.alpha.shape[1]

    @property
    def channels(self) -> int:
        return self.features.shape[2]


@dataclass(frozen=True)
class RenderOptions:
    lambda_th: float = 0.01
    sigma_dep: float = 5.0
    background: object = None
    image_size: tuple | None = None

    def __post_init__(self):
        if not 0.0 < self.lambda_th < 1.0:
            raise ContractViolation("lambda_th must be in (0, 1)")
        if self.sigma_dep < 0.0:
            raise ContractViolation("sigma_dep must be >= 0")
        # render.py:56-63: background flattened to fp64, image_size positive
        if self.background is not None:
            bg = np.asarray(self.background, dtype=np.float64).reshape(-1)
            object.__setattr__(self, "background", bg)
        if self.image_size is not None:
            w, h = self.image_size
            if w < 1 or h < 1:
                raise ContractViolation("image_size must be positive")


@dataclass(frozen=True)
class VoxelSet:
    resolution: int
    bounds: object
    cells: np.ndarray

    def __len__(self) -> int:
        return self.cells.shape[0]


@dataclass
class FLUT:
    data: np.ndarray
    degree: int
    channels: int

    def __len__(self) -> int:
        return self.data.shape[0]

    @property
    def densities(self) -> np.ndarray:
        return self.data[:, -1]


@dataclass(frozen=True)
class RigidTransform:
    rotation: np.ndarray
    translation: np.ndarray


@dataclass(frozen=True)
class Skeleton:
    names: tuple
    parents: np.ndarray
    bind_local: tuple


@dataclass(frozen=True)
class SkinWeights:
    joint_indices: np.ndarray
    weights: np.ndarray

    @property
    def n_voxels(self) -> int:
        return self.joint_indices.shape[0]


@dataclass(frozen=True)
class CharacterAsset:
    voxels: object
    flut: object
    skeleton: object = None
    weights: object = None

    @property
    def rigged(self) -> bool:
        return self.skeleton is not None


# factories (rebound by install.py to the reference's classes)
FACTORIES = {
    "VoxelOctree": VoxelOctree,
    "WarpResult": WarpResult,
    "CollisionResolution": CollisionResolution,
    "FrameBuffers": FrameBuffers,
    "Bounds": Bounds,
    "VoxelSet": VoxelSet,
    "FLUT": FLUT,
    "RigidTransform": RigidTransform,
    "Skeleton": Skeleton,
    "SkinWeights": SkinWeights,
    "CharacterAsset": CharacterAsset,
}


def make(kind: str, **kw):
    return FACTORIES[kind](**kw)
