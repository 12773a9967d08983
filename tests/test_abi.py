"""The C-ABI library loads without a GPU and exports every symbol include/flowprefill.h
declares; without a device the context constructor fails loudly (no CPU fallback)."""

import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "flowprefill.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|const char\*)\s+(fp_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_16603_b200 import _lib, build

    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    from paper_2602_16603_b200 import _lib

    names = declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.exported_symbols())


def test_error_path_without_device(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2602_16603_b200 import _lib

    cfg = _lib.ModelCfg(4, 512, 4, 2, 128, 1536, 8192, 1024, 1e4, 1e-5)
    h = C.c_void_p()
    rc = lib.fp_ctx_create(0, C.byref(cfg), 0, 1, None, 8, 128, C.byref(h))
    assert rc < 0
    assert lib.fp_last_error()
    with pytest.raises(_lib.NativeError):
        _lib.check(rc, "fp_ctx_create")


def test_argument_validation(lib):
    from paper_2602_16603_b200 import _lib

    cfg = _lib.ModelCfg(4, 512, 4, 2, 64, 1536, 8192, 1024, 1e4, 1e-5)  # head_dim 64
    h = C.c_void_p()
    assert lib.fp_ctx_create(0, C.byref(cfg), 0, 1, None, 8, 128, C.byref(h)) == -1
    assert b"head_dim" in lib.fp_last_error()
    cfg.head_dim = 128
    assert lib.fp_ctx_create(0, C.byref(cfg), 0, 3, None, 8, 128, C.byref(h)) == -1  # 2 kv heads
    assert b"tp_size" in lib.fp_last_error()
    assert lib.fp_ctx_create(0, C.byref(cfg), 2, 2, None, 8, 128, C.byref(h)) == -1  # rank >= size
    assert lib.fp_ctx_create(0, C.byref(cfg), 0, 2, C.c_void_p(1), 8, 128, C.byref(h)) == -1
    assert b"nccl_comm" in lib.fp_last_error()
    assert lib.fp_ctx_create(0, C.byref(cfg), 0, 1, None, 8, 64, C.byref(h)) == -1
