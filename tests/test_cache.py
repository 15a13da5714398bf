"""Host side of the kernel-contract device cache (no GPU needed): the
content digest that keys cached device FLUTs and trees covers every byte,
does not depend on the hashing thread count, and the cache policy knob."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from paper_2202_05628_b200 import _lib, build_lib


@pytest.fixture(scope="module")
def lib():
    build_lib.build()
    return _lib.load_library()


def digest(lib, a, threads):
    a = np.ascontiguousarray(a)
    out = (C.c_uint64 * 2)()
    assert lib.artemis_host_checksum(a.ctypes.data, a.nbytes, threads, out) == 0
    return (out[0], out[1])


def test_thread_count_independent(lib):
    a = np.random.default_rng(0).normal(size=(3_000_003,))  # 24 MB, ragged tail block
    ref = digest(lib, a, 1)
    for t in (2, 3, 8, 16):
        assert digest(lib, a, t) == ref


@pytest.mark.parametrize("nbytes", [0, 1, 7, 8, 31, 33, 65536, 65537, 200_001])
def test_every_byte_counts(lib, nbytes):
    rng = np.random.default_rng(nbytes)
    a = rng.integers(0, 256, size=nbytes, dtype=np.uint8)
    base = digest(lib, a, 4)
    assert digest(lib, a.copy(), 4) == base
    for i in sorted({0, nbytes // 2, nbytes - 1} - {-1}):
        if nbytes == 0:
            break
        b = a.copy()
        b[i] ^= 1
        assert digest(lib, b, 4) != base, i
    if nbytes:
        assert digest(lib, a[:-1], 4) != base  # length is part of the digest


def test_single_ulp_edit_of_a_large_flut(lib):
    fl = np.random.default_rng(1).normal(size=(200_000, 145))
    base = digest(lib, fl, 8)
    fl[123_457, 144] = np.nextafter(fl[123_457, 144], np.inf)
    assert digest(lib, fl, 8) != base


def test_content_key_and_policy(lib):
    from paper_2202_05628_b200 import kernels as K

    a = np.arange(1000, dtype=np.float64)
    k1 = K.content_key(a)
    assert k1 == K.content_key(a.copy())
    b = a.copy()
    b[999] += 1
    assert K.content_key(b) != k1
    assert K.content_key(a.astype(np.float32)) != k1  # dtype is part of the key
    K.set_cache_policy("identity")
    try:
        assert K.content_key(a)[0] == "id"
        assert K.content_key(a) != K.content_key(a.copy())  # another buffer
    finally:
        K.set_cache_policy("content")
    with pytest.raises(ValueError):
        K.set_cache_policy("sampled")


def test_host_widen_rect(lib):
    """artemis_host_widen_f32: exact fp32 -> fp64 of a row-strided block
    (the per-frame API's FrameBuffers.features readout)."""
    rng = np.random.default_rng(2)
    src = rng.normal(size=(300, 700)).astype(np.float32)
    dst = np.zeros((300, 900), dtype=np.float64)
    r0, c0, rows, cols = 17, 40, 250, 600
    off_s = r0 * 700 + c0
    off_d = r0 * 900 + c0 + 100
    assert lib.artemis_host_widen_f32(src.ctypes.data + 4 * off_s, rows, cols, 700,
                                      dst.ctypes.data + 8 * off_d, 900, 8) == 0
    want = np.zeros_like(dst)
    want[r0:r0 + rows, c0 + 100:c0 + 100 + cols] = src[r0:r0 + rows, c0:c0 + cols]
    assert np.array_equal(dst, want)
