"""Native host FK (artemis_host_pose_tables, csrc/hostfk.cu) against the
numpy restatement (kinematics.pose_tables) and the reference's own tables.

The native path is the frame stream's per-frame FK (FramePipeline.tables);
it must give the same doubles as the reference's numpy FK
(rigging.py:228-247, 343-347) -- bit for bit, signed zeros included. CPU
only: the library is loaded without a device."""
from __future__ import annotations

import numpy as np

from paper_2202_05628_b200 import kinematics as K
from paper_2202_05628_b200 import synthetic as S


def _same(a: K.PoseTables, b: K.PoseTables) -> bool:
    return all(x.tobytes() == y.tobytes() for x, y in ((a.delta_mats, b.delta_mats),
                                                        (a.delta_quats, b.delta_quats),
                                                        (a.rot_inv, b.rot_inv)))


def test_native_agrees_with_numpy_on_this_host():
    assert K.NativePoseTables.agrees()


def test_native_equals_reference_fixture(golden_mini):
    sc = S.make_scene("c0", resolution=64, image=(64, 64))
    t = K.NativePoseTables(sc.rig)(K.PoseSpec.make(sc.poses[0]))
    assert np.array_equal(t.delta_mats, golden_mini["delta_mats"])
    assert np.array_equal(t.delta_quats, golden_mini["delta_quats"])
    assert np.array_equal(t.rot_inv, golden_mini["rot_inv"])


def test_native_equals_numpy_on_config_sequences():
    for name in ("c3", "c4"):
        sc = S.make_scene(name, frames=16)
        canon = K.canonical_globals(sc.rig)
        nat = K.NativePoseTables(sc.rig, canon)
        for f in range(16):
            pose = K.PoseSpec.make(sc.poses[f])
            assert _same(K.pose_tables(sc.rig, pose, canonical=canon), nat(pose)), (name, f)


def test_native_edge_poses():
    rng = np.random.default_rng(7)
    sc = S.make_scene("c0", resolution=64, image=(64, 64))
    canon = K.canonical_globals(sc.rig)
    nat = K.NativePoseTables(sc.rig, canon)
    J = sc.rig.n_joints
    poses = [
        K.PoseSpec.make(np.zeros((J, 3))),                                  # canonical
        K.PoseSpec.make(np.full((J, 3), np.pi)),                            # wrap boundary
        K.PoseSpec.make(np.full((J, 3), -0.0)),                             # signed zeros
        K.PoseSpec.make(rng.uniform(-1e-9, 1e-9, (J, 3))),                  # tiny angles
        K.PoseSpec.make(rng.uniform(-50, 50, (J, 3)), [0.0, 0.0, 0.0, 1.0], [1e6, -1e6, 0.5]),
    ]
    for pose in poses:
        assert _same(K.pose_tables(sc.rig, pose, canonical=canon), nat(pose))


def test_native_rejects_bad_input():
    import pytest

    from paper_2202_05628_b200.errors import ContractViolation

    sc = S.make_scene("c0", resolution=64, image=(64, 64))
    nat = K.NativePoseTables(sc.rig)
    with pytest.raises(ContractViolation):
        nat(K.PoseSpec.make(np.zeros((sc.rig.n_joints + 1, 3))))
    with pytest.raises(ContractViolation):  # zero global quaternion
        nat(K.PoseSpec.make(np.zeros((sc.rig.n_joints, 3)), [0.0, 0.0, 0.0, 0.0]))
