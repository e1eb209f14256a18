"""CPU checks of the C-ABI library: it loads, exports exactly what include/lfgpu.h
declares, and fails loudly (no CPU fallback) when no GPU is visible."""
import ctypes
import os
import re

import numpy as np
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
    assert lfgpu._lib.lfg_abi_version() == 5
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


def test_per_sample_generator_is_mt19937_64(lfgpu, oracle):
    """The product's lazily seeded generator equals std::mt19937_64 (the oracle's
    restatement, itself pinned to libstdc++) across the lazy / library boundary at
    output 156, for the experiment.cpp:163 per-id seeding."""
    for seed, sid in ((1, 0), (1, 12345), (7, (1 << 40) + 3), (0, 2**64 - 2)):
        got = lfgpu.rng_outputs(seed, sid, 400)
        s0 = (seed ^ ((0x9E3779B97F4A7C15 * (sid + 1)) & (2**64 - 1))) & (2**64 - 1)
        assert np.array_equal(got, oracle.mt64(s0, 400))


def test_ctypes_structs_match_the_header(lfgpu, tmp_path):
    """Every ctypes mirror in lfgpu.py has the C layout of include/lfgpu.h: size and
    field offsets, checked against gcc's offsetof."""
    import subprocess
    structs = {"lfg_op": lfgpu.Op, "lfg_sample_desc": lfgpu.SampleDesc, "lfg_config": lfgpu.Config,
               "lfg_counters": lfgpu.Counters, "lfg_run_config": lfgpu.RunConfig,
               "lfg_run_report": lfgpu.RunReport}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "lfgpu.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.dirname(lfgpu.HEADER_PATH), str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
