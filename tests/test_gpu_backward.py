"""GPU parity of backward_rays (training gradients, _core.pyx:661-755)
against the reference's own output (tests/golden/backward.npz) and the CPU
oracle, through the drop-in `kernels.backward_rays` and the C ABI.

Tolerances: the per-hit terms use CUDA's exp (<= 1 ulp from glibc's), so
fp64 gradients agree to ~1e-15 relative; we require 1e-12 x max|grad|
(the reference's own fast-mode bar is 1e-9, test_backend.py:218-232). The
float32 instantiation must agree within 1e-6 x max|grad| (one float ulp on
a few entries). Untouched rows are exactly zero, and the result is
bit-reproducible run to run (no atomics on gradient values).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2202_05628_b200 import kernels as K
from paper_2202_05628_b200 import synthetic as S

pytestmark = pytest.mark.gpu

TOL64, TOL32 = 1e-12, 1e-6


def close(got, want, tol):
    scale = max(np.abs(want).max(), 1e-300)
    err = np.abs(np.asarray(got, np.float64) - np.asarray(want, np.float64)).max()
    assert err <= tol * scale, (err, scale)


def kernel_args(k):
    return (k["scene_fit_off"], k["scene_fit_idx"], k["scene_fit_t0"], k["scene_fit_t1"],
            k["scene_dirs"], k["scene_rot_index"], k["scene_rot_inv"])


@pytest.fixture(scope="module")
def mini():
    return S.make_scene("c0", resolution=64, image=(64, 64))


class TestGolden:
    def test_kernel_scene_fp64(self, golden_kernels, golden_backward):
        k, b = golden_kernels, golden_backward
        g = K.backward_rays(*kernel_args(k), k["scene_flut"], b["k_dldf"], b["k_dlda"], 2, 3)
        assert g.dtype == np.float64 and g.shape == b["k_grad64"].shape
        close(g, b["k_grad64"], TOL64)
        assert np.array_equal(g == 0, b["k_grad64"] == 0)

    def test_kernel_scene_float32_instantiation(self, golden_kernels, golden_backward):
        k, b = golden_kernels, golden_backward
        g = K.backward_rays(*kernel_args(k), k["scene_flut"].astype(np.float32),
                            b["k_dldf"].astype(np.float32), b["k_dlda"].astype(np.float32), 2, 3,
                            True, 1)
        assert g.dtype == np.float32
        close(g, b["k_grad32"], TOL32)

    def test_posed_scene_trace(self, golden_mini, golden_backward, mini):
        m, b = golden_mini, golden_backward
        common = (m["fit_off"], m["fit_idx"], m["fit_t0"], m["fit_t1"], m["rays_d"],
                  m["warp_rotation_joint"], m["rot_inv"])
        g = K.backward_rays(*common, mini.flut64(), b["m_dldf"], b["m_dlda"], mini.degree,
                            mini.channels)
        close(g, b["m_grad64"], TOL64)
        touched = np.zeros(len(g), bool)
        touched[m["fit_idx"]] = True
        assert not g[~touched].any()
        g32 = K.backward_rays(*common, mini.flut32, b["m_dldf"].astype(np.float32),
                              b["m_dlda"].astype(np.float32), mini.degree, mini.channels)
        close(g32, b["m_grad32"], TOL32)

    def test_deterministic_and_fast_mode_bit_identical(self, golden_kernels, golden_backward):
        k, b = golden_kernels, golden_backward
        args = (*kernel_args(k), k["scene_flut"], b["k_dldf"], b["k_dlda"], 2, 3)
        g1 = K.backward_rays(*args, True, 1)
        g2 = K.backward_rays(*args, True, 1)
        g3 = K.backward_rays(*args, False, 8)
        assert np.array_equal(g1, g2) and np.array_equal(g1, g3)


class TestOracle:
    def test_configs0_full_frame_trace(self):
        """configs[0] (128^3, 256^2, C = 16): the GPU's own forward_fit trace
        of a posed frame, gradients vs the oracle on the same trace."""
        from paper_2202_05628_b200 import kinematics as KM
        sc = S.make_scene("c0")
        tables = KM.pose_tables(sc.rig, KM.PoseSpec.make(sc.poses[0]))
        fr = oracle.render_frame(sc, tables, sc.cameras[0][0])
        codes, fidx, root, left, right, bmin, bsize = fr["tree"]
        og, dg, dw = fr["origins_g"], fr["dirs_g"], fr["dirs_w"]
        rot_index, rot_inv = fr["rotation_joint"], tables.rot_inv
        flut = sc.flut64()
        F, A, off, hi, h0, h1 = K.forward_fit(codes, fidx, root, left, right, bmin, bsize, og,
                                              dg, dw, 0.0, np.inf, flut, rot_index, rot_inv,
                                              sc.degree, sc.channels)
        rng = np.random.default_rng(5)
        n = og.shape[0]
        dldf = np.sign(rng.normal(size=(n, sc.channels))) / n
        dlda = np.sign(rng.normal(size=n)) / n
        args = (off, hi, h0, h1, dw, rot_index, rot_inv)
        g = K.backward_rays(*args, flut, dldf, dlda, sc.degree, sc.channels)
        want = oracle.backward_rays(*args, flut, dldf, dlda, sc.degree, sc.channels)
        close(g, want, TOL64)
        g32 = K.backward_rays(*args, sc.flut32, dldf.astype(np.float32),
                              dlda.astype(np.float32), sc.degree, sc.channels)
        want32 = oracle.backward_rays(*args, sc.flut32, dldf, dlda, sc.degree, sc.channels)
        close(g32, want32, TOL32)

    @pytest.mark.parametrize("degree,channels", [(0, 1), (1, 5), (3, 7), (4, 33)])
    def test_degrees_channels_and_ragged_traces(self, golden_kernels, degree, channels):
        """Every SH degree, channel counts around the warp width (the kernel
        scene's ragged trace, a synthetic FLUT)."""
        k = golden_kernels
        off, hi = k["scene_fit_off"], k["scene_fit_idx"]
        n_flut = int(k["scene_flut"].shape[0])
        rng = np.random.default_rng(degree * 100 + channels)
        width = (degree + 1) ** 2 * channels + 1
        flut = rng.uniform(-0.5, 1.0, size=(n_flut, width))
        flut[:, -1] = np.abs(flut[:, -1]) * 3
        n = off.size - 1
        dldf = rng.normal(size=(n, channels))
        dlda = rng.normal(size=n)
        args = (off, hi, k["scene_fit_t0"], k["scene_fit_t1"], k["scene_dirs"],
                k["scene_rot_index"], k["scene_rot_inv"])
        g = K.backward_rays(*args, flut, dldf, dlda, degree, channels)
        close(g, oracle.backward_rays(*args, flut, dldf, dlda, degree, channels), TOL64)

    def test_empty_trace_and_no_rays(self, golden_kernels):
        k = golden_kernels
        flut = k["scene_flut"]
        z = np.zeros(0)
        g = K.backward_rays(np.zeros(4, np.int64), np.zeros(0, np.int64), z, z,
                            np.zeros((3, 3)), k["scene_rot_index"], k["scene_rot_inv"], flut,
                            np.zeros((3, 3)), np.zeros(3), 2, 3)
        assert g.shape == flut.shape and not g.any()
        g = K.backward_rays(np.zeros(1, np.int64), np.zeros(0, np.int64), z, z,
                            np.zeros((0, 3)), k["scene_rot_index"], k["scene_rot_inv"], flut,
                            np.zeros((0, 3)), np.zeros(0), 2, 3)
        assert not g.any()
