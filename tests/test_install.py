"""The installer rebinds the reference package's hot path by name (CPU; the
reference is only present in the build container)."""

from __future__ import annotations

import os
import sys

import pytest

REF = os.environ.get("ARTEMIS_REF_ROOT", "/root/reference") + "/pkg/src"


@pytest.fixture()
def animvox():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    sys.path.insert(0, REF)
    os.environ.setdefault("ANIMVOX_BACKEND", "pure")
    import animvox.backend  # noqa: F401
    import animvox.render
    import animvox.rigging
    import animvox.volume

    yield sys.modules["animvox"]
    sys.path.remove(REF)


def test_install_rebinds_and_restores(animvox):
    import animvox.render as R
    import animvox.rigging as RG
    import animvox.volume as V

    from paper_2202_05628_b200 import install, kernels, pipeline, types

    orig = (R.kernels, RG.warp_voxels, V.build_octree, R.render_view)
    done = install.install("animvox")
    try:
        assert ("render", "kernels") in done and ("volume", "build_octree") in done
        assert R.kernels is kernels and V.kernels is kernels
        assert RG.warp_voxels is pipeline.warp_voxels
        assert R.warp_voxels is pipeline.warp_voxels
        assert R.resolve_collisions is pipeline.resolve_collisions
        assert V.build_octree is pipeline.build_octree and R.build_octree is pipeline.build_octree
        assert R.render_view is pipeline.render_view
        assert R.timed_render_frame is pipeline.timed_render_frame
        assert types.FACTORIES["VoxelOctree"] is V.VoxelOctree
        assert types.FACTORIES["WarpResult"] is RG.WarpResult
        import animvox.errors as E

        assert pipeline.DuplicateMortonError is E.DuplicateMortonError
    finally:
        install.uninstall("animvox")
    assert (R.kernels, RG.warp_voxels, V.build_octree, R.render_view) == orig
    assert types.FACTORIES["VoxelOctree"] is types.VoxelOctree
