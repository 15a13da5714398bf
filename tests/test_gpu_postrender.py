"""GPU parity of the post-render frame-buffer step:
device over_background / composite / straight RGBA / RGBA8 against the
reference's own outputs (tests/golden/post.npz) and the oracle, bit for bit,
with float and double alpha/depth maps, and on a rendered frame."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2202_05628_b200 import compositing as CP
from paper_2202_05628_b200 import kinematics as KM
from paper_2202_05628_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).cuda()


@pytest.mark.parametrize("maps64", [False, True])
def test_against_reference_golden(golden_post, maps64):
    g = golden_post
    mt = np.float64 if maps64 else np.float32
    F = dev(g["F"].reshape(-1, 3), np.float32)
    A = dev(g["A"].reshape(-1), mt)
    D = dev(g["D"].reshape(-1), mt)
    over = CP.over_background(F, A, g["color"]).cpu().numpy()
    assert np.array_equal(over, g["over"].reshape(-1, 3))
    comp = CP.composite(F, A, D, g["bg_color"].reshape(-1, 3), g["bg_depth"].reshape(-1))
    assert np.array_equal(comp.cpu().numpy(), g["composite"].reshape(-1, 3))
    assert np.array_equal(CP.straight_rgba(F, A).cpu().numpy(), g["rgba"].reshape(-1, 4))
    assert np.array_equal(CP.rgba8(F, A).cpu().numpy(), g["rgba8"].reshape(-1, 4))


def test_on_rendered_frame():
    """A 3-channel posed frame straight out of the frame pipeline."""
    from paper_2202_05628_b200.frame import FramePipeline

    sc = S.make_scene("c0", resolution=64, channels=3, image=(72, 56))
    fp = FramePipeline.from_scene(sc)
    pose = KM.PoseSpec.make(sc.poses[0])
    cam = sc.cameras[0][0]
    rng = np.random.default_rng(3)
    for maps64 in (False, True):
        F, A, D = fp.run(pose, cam, graph=False, maps64=maps64)
        torch.cuda.synchronize()
        Fh, Ah, Dh = F.cpu().numpy(), A.cpu().numpy(), D.cpu().numpy()
        n = Ah.size
        bgc = rng.uniform(size=(n, 3))
        bgd = np.where(rng.uniform(size=n) < 0.5, rng.uniform(1.5, 4.0, n), np.inf)
        assert np.array_equal(CP.composite(F, A, D, bgc, bgd).cpu().numpy(),
                              oracle.composite(Fh, Ah, Dh, bgc, bgd))
        assert np.array_equal(CP.over_background(F, A, [0.1, 0.2, 0.3]).cpu().numpy(),
                              oracle.over_background(Fh, Ah, [0.1, 0.2, 0.3]))
        assert np.array_equal(CP.rgba8(F, A).cpu().numpy(), oracle.rgba8(Fh, Ah))
    fp.close()


def test_contract_errors():
    from paper_2202_05628_b200.errors import ContractViolation

    F = torch.zeros((4, 5), dtype=torch.float32, device="cuda")
    A = torch.zeros(4, dtype=torch.float32, device="cuda")
    with pytest.raises(ContractViolation):
        CP.over_background(F, A, [0.0, 0.0])
    with pytest.raises(ContractViolation):
        CP.rgba8(F, A)
