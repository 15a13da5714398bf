"""GPU side of .nvo ingestion: leaves decoded and
scattered on the device, the FLUT split on the device, the drop-in
load_asset returning the reference's arrays bit for bit (digests from the
reference's own load_asset), the permutation check on the device, and a
frame rendered from the device-resident asset equal to one rendered from
the original scene."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from paper_2202_05628_b200 import assetio as AIO
from paper_2202_05628_b200 import kinematics as KM
from paper_2202_05628_b200 import synthetic as S
from test_assetio import corruptions, digest, encode

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["rig", "still"])
def test_load_asset_matches_reference(golden_asset, case):
    g = golden_asset
    asset = AIO.load_asset(encode(case == "rig"))
    assert digest(asset.voxels.cells) == str(g[f"{case}_sha_cells"])
    assert digest(asset.flut.data) == str(g[f"{case}_sha_flut"])
    assert digest(asset.voxels.bounds.lo) == str(g[f"{case}_sha_lo"])
    assert asset.voxels.resolution == int(g[f"{case}_resolution"])
    if case == "rig":
        sk = asset.skeleton
        assert "|".join(sk.names) == str(g["rig_names"])
        assert digest(sk.parents) == str(g["rig_sha_parents"])
        bind = np.array([[*b.rotation, *b.translation] for b in sk.bind_local])
        assert digest(bind) == str(g["rig_sha_bind"])
        assert digest(asset.weights.joint_indices) == str(g["rig_sha_joint_idx"])
        assert digest(asset.weights.weights) == str(g["rig_sha_weights"])
    else:
        assert asset.skeleton is None and asset.weights is None


def test_device_permutation_check(golden_asset):
    data = encode(True)
    sc = S.make_scene("c0", resolution=64, image=(64, 64), with_flut=False)
    width = (sc.degree + 1) ** 2 * sc.channels + 1
    bad = corruptions(data, sc.cells.shape[0], width)["not_permutation"]
    with pytest.raises(Exception) as ei:
        AIO.load_asset(bad)
    assert type(ei.value).__name__ == str(golden_asset["err_not_permutation"])


def test_render_from_loaded_asset_equals_scene():
    """The device-resident loaded character renders the same frame as the
    scene it was saved from, with the container's precision (FLUT and skin
    weights stored at f32, assetio.py:64 / :154)."""
    from paper_2202_05628_b200 import pipeline as P
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c0", resolution=64, image=(64, 64))
    asset = AIO.load_asset(encode(True))
    fp = P.DEVICE_ASSETS.get(asset)  # adopted at load: no re-upload
    assert fp is not None
    pose = KM.PoseSpec.make(sc.poses[0])
    cam = sc.cameras[0][0]
    F1, A1, D1 = [x.clone() for x in fp.run(pose, cam, graph=False)]
    ref = FramePipeline(sc.cells, sc.skin_idx, sc.skin_w.astype(np.float32).astype(np.float64),
                        sc.flut32, sc.degree, sc.channels, sc.resolution, sc.lo, sc.hi,
                        rig=sc.rig)
    F2, A2, D2 = [x.clone() for x in ref.run(pose, cam, graph=False)]
    ref.stream.synchronize()
    fp.stream.synchronize()
    assert (F1 == F2).all() and (A1 == A2).all() and (D1 == D2).all()
    fb = P.render_frame(asset, pose, cam)
    assert fb.features.shape == (64, 64, sc.channels)
    ref.close()
    P.DEVICE_ASSETS.clear()
