"""C-ABI surface checks that run without a GPU: libartemis.so loads, exports
every function include/artemis.h declares, and the product refuses to run
(no CPU fallback) when no sm_100 device is visible."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest
import torch

from paper_2202_05628_b200 import _lib, build_lib
from paper_2202_05628_b200.errors import ExtensionMissing

HEADER = os.path.join(build_lib.REPO, "include", "artemis.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(artemis_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    build_lib.build()
    return _lib.load_library()


def test_header_declares_functions():
    names = declared_functions()
    assert "artemis_render_rays" in names and "artemis_frame_run" in names
    assert len(names) >= 25


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    assert sorted(_lib.EXPORTS) == declared_functions()


def test_status_strings(lib):
    assert lib.artemis_status_string(0) == b"ok"
    assert b"duplicate" in lib.artemis_status_string(4)
    assert lib.artemis_version().startswith(b"libartemis")


def test_built_for_sm100a():
    out = os.popen(f"cuobjdump --list-elf {build_lib.LIB} 2>&1").read()
    assert "sm_100a" in out


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU refusal")
def test_no_cpu_fallback():
    from paper_2202_05628_b200 import kernels

    with pytest.raises(ExtensionMissing):
        kernels.morton_encode(np.array([[1, 2, 3]]))


def test_argument_errors_need_no_device(lib):
    # a null-pointer call is rejected before any CUDA work is enqueued
    assert lib.artemis_morton_encode(None, 5, None, None, None) == _lib.ERR_ARG
    assert lib.artemis_build_tree(ctypes.c_void_p(1), 0, None, None, None, None, None,
                                  None) == _lib.ERR_EMPTY
