"""C-ABI boundary checks that need no GPU.

* libtokenselect.so (sm_100a build) loads and exports every entry point that
  include/tokenselect.h declares — the symbol set a reference-side FFI binding
   would bind;
* the exported symbol set is exactly the header's (nothing undeclared leaks);
* EngineConfig defaults and validation (attention.hpp:13-22, attention.cpp:10-19)
  run host-side;
* without a CUDA device every compute entry point fails loudly with
  TS_CUDA_ERROR (there is no CPU fallback);
* the .so carries sm_100a SASS only, and its kernels use the TMA bulk-copy and
  tensor-core instructions the design relies on.
"""
import ctypes as C
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tokenselect.h")
LIB = os.path.join(ROOT, "paper_2411_02886_b200", "_build", "libtokenselect.so")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(ts_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2411_02886_b200 import build

        build.build()
    return C.CDLL(LIB)


def test_header_declares_the_boundary():
    names = header_functions()
    for must in ("ts_pool_create", "ts_pool_append_kv", "ts_score_paged", "ts_select", "ts_select_for_chunk",
                 "ts_sparse_attend", "ts_engine_decode", "ts_engine_prefill", "ts_last_error"):
        assert must in names
    assert len(names) >= 40


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_no_undeclared_exports():
    nm = shutil.which("nm")
    if not nm:
        pytest.skip("nm not available")
    out = subprocess.run([nm, "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = sorted({ln.split()[-1] for ln in out.splitlines() if " T " in ln and ln.split()[-1].startswith("ts_")})
    assert exported == header_functions()


def test_python_binding_covers_header():
    from paper_2411_02886_b200._native import SIGNATURES

    assert sorted(SIGNATURES) == header_functions()


def test_config_defaults_and_validation(lib):
    from paper_2411_02886_b200._native import EngineConfig, TsStatus

    cfg = EngineConfig()
    lib.ts_engine_config_default(C.byref(cfg))
    assert (cfg.k, cfg.n_local, cfg.n_init, cfg.chunk_size, cfg.theta) == (2048, 512, 128, 512, 0.9)
    assert (cfg.num_heads, cfg.num_kv_heads, cfg.head_dim, cfg.block_size, cfg.selection_method) == (8, 8, 64, 64, 2)
    lib.ts_engine_config_validate.argtypes = [C.c_void_p]
    lib.ts_last_error.restype = C.c_char_p
    assert lib.ts_engine_config_validate(C.byref(cfg)) == TsStatus.OK
    cfg.num_kv_heads = 3
    assert lib.ts_engine_config_validate(C.byref(cfg)) == TsStatus.INVALID_ARGUMENT
    assert b"multiple" in lib.ts_last_error()
    cfg.num_kv_heads, cfg.chunk_size = 8, 0
    assert lib.ts_engine_config_validate(C.byref(cfg)) == TsStatus.INVALID_ARGUMENT
    cfg.chunk_size, cfg.block_size = 512, 0
    assert lib.ts_engine_config_validate(C.byref(cfg)) == TsStatus.INVALID_ARGUMENT


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device failure path")
def test_no_cpu_fallback(lib):
    from paper_2411_02886_b200._native import TsStatus

    lib.ts_last_error.restype = C.c_char_p
    h = C.c_void_p()
    rc = lib.ts_pool_create(C.c_size_t(64), C.c_size_t(1), C.c_size_t(1), C.c_size_t(4), C.byref(h))
    assert rc == TsStatus.CUDA_ERROR
    assert b"no CUDA device" in lib.ts_last_error()


def test_sm100a_sass_only():
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", LIB], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs
    sass = subprocess.run([cuobjdump, "-sass", LIB], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass, "TMA bulk copies (cp.async.bulk) expected in the decode kernel"
    assert "HMMA" in sass or "UTCHMMA" in sass or "UTCQMMA" in sass, "tensor-core scan expected"
