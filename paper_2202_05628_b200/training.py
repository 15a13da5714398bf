"""The training iteration on the device.

The reference's fit loop (animvox/fit.py:404-540) runs, per iteration:
forward_fit on a ray batch (full integration + CSR trace), the L1 loss
gradients sign(f - gt) / n (fit.py:486-488), backward_rays (the FLUT
gradient, :108-146), the collision-pair (VRT) term added with np.add.at
(:494-501), SparseAdam on the touched rows (:308-330) and the density clamp
(volume.py:166-167). `DeviceTrainer.step` does all of it with the FLUT, the
Adam moments, the trace and the gradient resident on the device; only the
batch's rays/targets go up and the loss comes back.

Given the same forward values, every update is the reference's arithmetic
bit for bit (fp64, numpy's evaluation order); the forward shades in fp32
(F within 1e-4 of the reference), which is the only difference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from . import kernels as K
from ._lib import check
from .device import empty, ptr, stream_handle, upload


class DeviceTrainer:
    """SparseAdam state (fit.py:308-330) on the device and one fit step."""

    def __init__(self, flut, degree: int, channels: int, *, learning_rate: float = 0.05,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 lambda_vrt: float = 0.01):
        fl = np.asarray(flut, dtype=np.float64)
        h = (int(degree) + 1) ** 2
        if fl.ndim != 2 or fl.shape[1] != h * int(channels) + 1:
            raise ValueError("flut must be (N, (degree+1)^2 * channels + 1)")
        self.degree, self.channels = int(degree), int(channels)
        self.params = upload(fl, np.float64)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.t = 0
        self.lr, self.beta1, self.beta2, self.eps = learning_rate, beta1, beta2, eps
        self.lambda_vrt = lambda_vrt

    @property
    def data(self) -> np.ndarray:
        return self.params.cpu().numpy()

    def shading(self, rot_index, rot_inv) -> K.DeviceShading:
        """Render layout of the current parameters (fp32 SH block + fp64
        density) without leaving the device."""
        L = _lib.lib()
        sh = K.DeviceShading.__new__(K.DeviceShading)
        n, width = self.params.shape
        sh.coef = empty((n, max(width - 1, 1)), np.float32)
        sh.sigma = empty(n, np.float64)
        check(L.artemis_flut_split_f64(ptr(self.params), n, width, ptr(sh.coef), ptr(sh.sigma),
                                       stream_handle()), "flut_split")
        sh.rot_index = upload(np.asarray(rot_index).reshape(-1), np.int32)
        sh.rot_inv = upload(np.asarray(rot_inv).reshape(-1, 9), np.float64)
        sh.view = _lib.Shading(ptr(sh.coef), ptr(sh.sigma), ptr(sh.rot_index), ptr(sh.rot_inv),
                               self.degree, self.channels, width - 1)
        return sh

    def step(self, tree, origins_g, dirs_g, dirs_w, gt_features, gt_alpha, rot_index, rot_inv,
             pairs=None):
        """One fit iteration on a ray batch. `tree` = (codes, flut_idx, root,
        left, right, box_min, box_size) of the batch's pose. Returns
        (l_rgba, l_vrt) as host floats."""
        L = _lib.lib()
        st = stream_handle()
        shade = self.shading(rot_index, rot_inv)
        dtree = K.DeviceTree(*tree, shade)
        rays = K.DeviceRays(origins_g, dirs_g, dirs_w, 0.0, np.inf)
        n = rays.n
        F, A, off, hit_idx, h0, h1 = K.forward_fit_device(dtree, shade, rays)
        gtf = upload(np.asarray(gt_features).reshape(n, self.channels), np.float64)
        gta = upload(np.asarray(gt_alpha).reshape(n), np.float64)
        dldf = empty((n, self.channels), np.float64)
        dlda = empty(n, np.float64)
        loss_rays = empty(n, np.float64)
        loss = empty(1, np.float64)
        check(L.artemis_l1_grads(ptr(F), ptr(A), ptr(gtf), ptr(gta), n, self.channels, ptr(dldf),
                                 ptr(dlda), ptr(loss_rays), ptr(loss), st), "l1_grads")
        grad = K.backward_rays_device(upload(off, np.int64), hit_idx, h0, h1, rays.dw,
                                      shade.rot_index, shade.rot_inv, self.params, dldf, dlda,
                                      self.degree, self.channels, True)
        n_rows, width = self.params.shape
        touched = torch.zeros(n_rows, dtype=torch.uint8, device=self.params.device)
        check(L.artemis_mark_touched(ptr(hit_idx), int(hit_idx.numel()), ptr(touched), st),
              "mark_touched")
        l_vrt = 0.0
        if pairs is not None and self.lambda_vrt > 0 and np.asarray(pairs).size:
            pr = upload(np.asarray(pairs, dtype=np.int64).reshape(-1, 2), np.int64)
            P = pr.shape[0]
            scale = self.lambda_vrt / (P * width)
            ws = torch.empty(L.artemis_vrt_workspace_bytes(P, n_rows), dtype=torch.uint8,
                             device=self.params.device)
            diff = self.params[pr[:, 0]] - self.params[pr[:, 1]]
            l_vrt = float(diff.abs().mean().item())  # loss_vrt (fit.py:71-80), reported
            check(L.artemis_vrt_grads(ptr(self.params), n_rows, width, ptr(pr), P, scale,
                                      ptr(grad), ptr(touched), ptr(ws), ws.numel(), st),
                  "vrt_grads")
        self.t += 1
        check(L.artemis_sparse_adam(ptr(self.params), ptr(self.m), ptr(self.v), ptr(grad),
                                    ptr(touched), n_rows, width, self.lr, self.beta1, self.beta2,
                                    self.eps, 1.0 - self.beta1 ** self.t,
                                    1.0 - self.beta2 ** self.t, st), "sparse_adam")
        return float(loss.item()) / n, l_vrt
