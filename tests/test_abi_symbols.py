"""CPU checks of the C-ABI boundary: the library builds, loads without a GPU and
exports every function include/dgnn.h declares (no compute calls here)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "dgnn.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(dgnn_[a-z0-9_]+)\s*\(", src))
    return sorted(n for n in names if not n.endswith("_fn"))


@pytest.fixture(scope="module")
def lib():
    from __graft_entry__ import _build_module
    build = _build_module()
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_four_calls():
    names = _declared()
    for n in ("dgnn_sample", "dgnn_build_cache", "dgnn_pack", "dgnn_assemble"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_exports_match_header():
    from paper_2405_05231_b200 import _abi
    assert sorted(_abi.EXPORTS) == _declared()


def test_library_is_sm100a():
    from __graft_entry__ import _build_module
    build = _build_module()
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_chunk_layout_is_host_arithmetic(lib):
    # dgnn_chunk_layout needs no GPU: reading c20 offsets
    import numpy as np
    from paper_2405_05231_b200 import _abi
    po = np.array([0, 3, 3, 12, 12, 13], np.int64)
    assert _abi.dgnn_chunk_layout(po, 400).tolist() == [0, 4096, 4096, 8192, 8192, 12288]


def test_errors_without_gpu_are_reported_not_raised(lib):
    from paper_2405_05231_b200 import _abi
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    with pytest.raises(_abi.DgnnError):
        _abi.Ctx(device=0, stream=None, torch_allocator=False) if False else _abi._check(
            _abi.load_library().dgnn_ctx_create(0, None, None, ctypes.byref(ctypes.c_void_p())), "dgnn_ctx_create")


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: a missing libdgnn.so is an ImportError, not a silent degradation."""
    import subprocess
    import sys
    code = ("import paper_2405_05231_b200._abi as a\n"
            "a._lib = None\n"
            "try:\n    a.load_library('/nonexistent/libdgnn.so')\nexcept ImportError as e:\n"
            "    print('IMPORT_ERROR', e)\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT).stdout
    assert "IMPORT_ERROR" in out and "no CPU fallback" in out
