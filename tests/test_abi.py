"""CPU checks of the C-ABI library: it loads, exports exactly what include/lfgpu.h
declares, and fails loudly (no CPU fallback) when no GPU is visible."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "lfgpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lfg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("lfg_open", "lfg_chain_create", "lfg_submit", "lfg_progress",
                     "lfg_seal_batch", "lfg_batch_release", "lfg_run_shard", "lfg_get_counters"):
        assert required in names


def test_library_exports_every_declared_symbol(lfgpu):
    lib = ctypes.CDLL(lfgpu.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"liblfgpu.so lacks {missing}"
    # and the Python binding binds all of them
    assert sorted(lfgpu.EXPORTED) == declared_functions()


def test_library_is_sm100a(lfgpu):
    out = os.popen(f"cuobjdump --list-elf {lfgpu.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_abi_version_and_defaults(lfgpu):
    assert lfgpu._lib.lfg_abi_version() == 4
    cfg = lfgpu.Config()
    lfgpu._lib.lfg_config_default(ctypes.byref(cfg))
    assert cfg.n_workers == 12 and cfg.batch_size == 24 and cfg.seed == 1


def test_no_cpu_fallback_without_gpu(lfgpu):
    if lfgpu.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(lfgpu.LfgError) as e:
        lfgpu.Context()
    assert e.value.code == lfgpu.ERR_CUDA


def test_errors_are_codes_not_crashes(lfgpu):
    with pytest.raises(lfgpu.LfgError) as e:
        lfgpu._check(lfgpu._lib.lfg_open(None, None))
    assert e.value.code == lfgpu.ERR_INVALID
    assert b"null" in lfgpu._lib.lfg_last_error()
