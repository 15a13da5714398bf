"""The .nvo container path, CPU side: the oracle's
encoder reproduces the reference's save_asset bytes, and the native host
half of the loader (header/extent validation, rig decode) reproduces the
reference's load_asset arrays and exception classes. The device half (leaf
decode + permutation check, FLUT split) is in test_gpu_assetio.py."""

from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np
import pytest

import oracle
from paper_2202_05628_b200 import _lib
from paper_2202_05628_b200 import assetio as AIO
from paper_2202_05628_b200 import build_lib
from paper_2202_05628_b200 import synthetic as S


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a))
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def lib():
    build_lib.build()
    return _lib.load_library()


def encode(rigged=True):
    sc = S.make_scene("c0", resolution=64, image=(64, 64))
    kw = {}
    if rigged:
        J = sc.rig.n_joints
        kw = dict(names=[f"j{j}" for j in range(J)], parents=sc.rig.parents,
                  bind=np.concatenate([sc.rig.bind_q, sc.rig.bind_t], axis=1),
                  joint_idx=sc.skin_idx, weights=sc.skin_w)
    return oracle.save_asset(sc.cells, sc.flut64(), sc.degree, sc.channels, sc.resolution,
                             sc.lo, sc.hi, **kw)


def corruptions(data: bytes, n: int, width: int) -> dict:
    """The same corruptions make_golden.asset_fixtures applies."""
    hs = 54
    flut_end = hs + 12 * n + 4 * width * n
    bad = bytearray(data)
    bad[hs + 8:hs + 12] = bad[hs + 20:hs + 24]
    return {
        "short_header": data[:40], "magic": b"NVO2" + data[4:],
        "version": data[:4] + (2).to_bytes(4, "little") + data[8:],
        "zero_count": data[:12] + (0).to_bytes(8, "little") + data[20:],
        "short_leaves": data[:hs + 12 * (n // 2)], "short_flut": data[:flut_end - 3],
        "not_permutation": bytes(bad),
        "rig_offset": data[:46] + (flut_end + 1).to_bytes(8, "little") + data[54:],
        "short_rig": data[:-2], "trailing": data + b"\0",
    }


@pytest.mark.parametrize("case", ["rig", "still"])
def test_encoder_reproduces_reference_bytes(golden_asset, case):
    data = encode(case == "rig")
    assert len(data) == int(golden_asset[f"{case}_size"])
    assert hashlib.sha256(data).hexdigest() == str(golden_asset[f"{case}_sha_bytes"])


def host_decode(lib, data: bytes):
    buf = np.frombuffer(data, np.uint8)
    info = _lib.AssetInfo()
    st = lib.artemis_asset_probe(buf.ctypes.data, buf.size, C.byref(info))
    if st:
        return st, None
    rig = _lib.AssetRig()
    st = lib.artemis_asset_decode_rig(buf.ctypes.data, buf.size, C.byref(info), C.byref(rig),
                                      None, None, None, None, None, None)
    if st or not info.rig_offset:
        return st, (info, None)
    J, K, n = rig.n_joints, rig.k_max, info.count
    parents = np.empty(J, np.int32)
    bind = np.empty((J, 7))
    raw = np.empty(max(rig.name_bytes, 1), np.uint8)
    offs = np.empty(J + 1, np.int32)
    jidx = np.empty((n, K), np.int32)
    w = np.empty((n, K))
    st = lib.artemis_asset_decode_rig(buf.ctypes.data, buf.size, C.byref(info), C.byref(rig),
                                      parents.ctypes.data, bind.ctypes.data, raw.ctypes.data,
                                      offs.ctypes.data, jidx.ctypes.data, w.ctypes.data)
    names = "|".join(raw.tobytes()[offs[j]:offs[j + 1]].decode() for j in range(J))
    return st, (info, dict(parents=parents, bind=bind, joint_idx=jidx, weights=w, names=names))


def test_native_header_and_rig_decode(lib, golden_asset):
    g = golden_asset
    st, (info, rig) = host_decode(lib, encode(True))
    assert st == 0
    assert info.resolution == int(g["rig_resolution"])
    assert digest(np.array(info.lo[:])) == str(g["rig_sha_lo"])
    assert digest(np.array(info.hi[:])) == str(g["rig_sha_hi"])
    for k in ("parents", "bind", "joint_idx", "weights"):
        assert digest(rig[k]) == str(g[f"rig_sha_{k}"]), k
    assert rig["names"] == str(g["rig_names"])
    st, (info, rig) = host_decode(lib, encode(False))
    assert st == 0 and rig is None


def test_host_detected_corruptions_raise_reference_classes(lib, golden_asset):
    data = encode(True)
    sc = S.make_scene("c0", resolution=64, image=(64, 64), with_flut=False)
    n = sc.cells.shape[0]
    width = (sc.degree + 1) ** 2 * sc.channels + 1
    for name, bad in corruptions(data, n, width).items():
        if name == "not_permutation":  # detected on the device
            continue
        st, _ = host_decode(lib, bad)
        assert st != 0, name
        with pytest.raises(Exception) as ei:
            AIO._raise_status(st)
        assert type(ei.value).__name__ == str(golden_asset[f"err_{name}"]), name
