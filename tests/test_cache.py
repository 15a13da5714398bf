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
