"""Post-render frame-buffer step on the device.

The consumers of a rendered frame -- solid-background compositing, the
depth-resolved blend over a rasterised scene (the hybrid-rendering use of
the depth buffer), the straight-alpha conversion and the 8-bit PNG
quantisation -- run on the frame while it is still on the GPU, so only the
final image crosses PCIe (4 bytes per pixel for an RGBA8 preview instead of
4(C+2)):

  over_background  FrameBuffers.over_background  animvox/render.py:98-104
  composite        composite                     animvox/render.py:366-382
  straight_rgba    frame_to_straight_rgba        animvox/assetio.py:265-275
  rgba8            + save_png/encode_png quantisation  assetio.py:209-245

Inputs are the device outputs of FramePipeline.run (F fp32 (n, C); alpha
and depth fp32, or fp64 with maps64). Results are bit-equal to the
reference's numpy expressions evaluated on the same values.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import check
from .device import empty, ptr, stream_handle, upload
from .errors import ContractViolation


def _maps64(A: torch.Tensor) -> int:
    if A.dtype == torch.float64:
        return 1
    if A.dtype == torch.float32:
        return 0
    raise ContractViolation("alpha/depth must be float32 or float64")


def _pixels(F: torch.Tensor, A: torch.Tensor) -> tuple[int, int]:
    n = A.numel()
    if F.dtype != torch.float32 or n == 0 and F.numel() != 0 or F.numel() % max(n, 1):
        raise ContractViolation("F must be fp32 (n_pix, C)")
    return n, (F.numel() // n if n else 1)


def over_background(F, A, color) -> torch.Tensor:
    """F + (1 - alpha) * color, (n_pix, C) fp64 on the device."""
    n, C = _pixels(F, A)
    col = np.asarray(color, dtype=np.float64).reshape(-1)
    if col.size != C:
        raise ContractViolation("background channel count mismatch")
    out = empty((n, C), np.float64)
    check(_lib.lib().artemis_over_background(ptr(F), ptr(A), _maps64(A), n, C,
                                             ptr(upload(col, np.float64)), ptr(out),
                                             stream_handle()), "over_background")
    return out


def composite(F, A, D, bg_color, bg_depth) -> torch.Tensor:
    """Depth-resolved blend over a rasterised scene; bg_color (n_pix, C) and
    bg_depth (n_pix) fp64 (device tensors or host arrays)."""
    n, C = _pixels(F, A)
    bc = bg_color if isinstance(bg_color, torch.Tensor) else upload(bg_color, np.float64)
    bd = bg_depth if isinstance(bg_depth, torch.Tensor) else upload(bg_depth, np.float64)
    if bc.numel() != n * C or bd.numel() != n or bc.dtype != torch.float64 \
            or bd.dtype != torch.float64:
        raise ContractViolation("composite buffer dimensions mismatch")
    if D.dtype != A.dtype:
        raise ContractViolation("alpha and depth must share a dtype")
    out = empty((n, C), np.float64)
    check(_lib.lib().artemis_composite(ptr(F), ptr(A), ptr(D), _maps64(A), n, C, ptr(bc),
                                       ptr(bd), ptr(out), stream_handle()), "composite")
    return out


def straight_rgba(F, A) -> torch.Tensor:
    """Straight-alpha RGBA (n_pix, 4) fp64 of a 3-channel frame."""
    n, C = _pixels(F, A)
    if C != 3:
        raise ContractViolation("expected (H, W, 3) features and (H, W) alpha")
    out = empty((n, 4), np.float64)
    check(_lib.lib().artemis_straight_rgba(ptr(F), ptr(A), _maps64(A), n, ptr(out),
                                           stream_handle()), "straight_rgba")
    return out


def rgba8(F, A) -> torch.Tensor:
    """The 8-bit straight-alpha RGBA a PNG stores, (n_pix, 4) uint8."""
    n, C = _pixels(F, A)
    if C != 3:
        raise ContractViolation("expected (H, W, 3) features and (H, W) alpha")
    out = torch.empty((n, 4), dtype=torch.uint8, device=F.device)
    check(_lib.lib().artemis_rgba8(ptr(F), ptr(A), _maps64(A), n, ptr(out), stream_handle()),
          "rgba8")
    return out
