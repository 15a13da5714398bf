"""Error categories of the drop-in boundary.

Mirrors the reference's exception taxonomy (`animvox/errors.py:5-66`) for
the errors the warp -> rebuild -> render path can raise, so callers that
catch by category keep working. When the reference package is importable
the installer (`install.py`) maps these onto the reference classes.
"""

from __future__ import annotations


class ArtemisError(Exception):
    category = "internal"


class ContractViolation(ArtemisError):
    """Caller broke a documented precondition (animvox ContractViolation)."""

    category = "contract"


class DuplicateMortonError(ArtemisError):
    """Octree build received colliding cells (animvox/volume.py:244-247)."""

    category = "duplicate-morton"


class EmptyWarpError(ArtemisError):
    """Every voxel warped outside the grid (animvox/render.py:170-171)."""

    category = "warp-empty"

    def __init__(self, dropped: int):
        self.dropped = dropped
        super().__init__(f"all {dropped} voxels warped out of bounds")


class AssetFormatError(ArtemisError):
    """Malformed .nvo container (animvox/errors.py AssetFormatError)."""

    category = "asset-format"


class TruncatedAssetError(AssetFormatError):
    category = "asset-truncated"


class MagicMismatchError(AssetFormatError):
    category = "asset-magic"


class CountMismatchError(AssetFormatError):
    category = "asset-count"


class DeviceError(ArtemisError):
    """The CUDA library reported a failure (status code from libartemis)."""

    category = "device"


class ExtensionMissing(ArtemisError, ImportError):
    """libartemis.so is not built or no CUDA device is present. The product
    path has no CPU fallback: this is raised instead of computing anything."""

    category = "extension-missing"
