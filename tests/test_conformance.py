"""Scheduling-semantics conformance: the reference's own doctest suites
(/root/reference/proj/tests/test_*.cpp, compiled from where they lie -- never
copied) built against THIS repo's reference-shaped headers (include/loadflow)
and host library (libloadflow_b200.so), with a doctest shim
(tests/conformance/doctest.h).  These are the known-answer tests for the
scheduling half of the hot path: timeout routing and resume (balancer),
fast-first eager batching, consumer idle accounting, the p75/p90 profiler,
queues, the virtual-time runtime and the workload generators.

CPU only.  Skipped where /root/reference is absent (the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
PKG = os.path.join(ROOT, "paper_2509_10712_b200")
BUILD = os.path.join(ROOT, "tests", "conformance", "build")

# hot-path suites + the adaptive scheduler and baselines
SUITES = ["core", "queue", "runtime", "balancer", "batcher", "trainer", "profiler", "workloads", "scheduler", "baselines"]

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                                reason="reference test sources not present")


@pytest.fixture(scope="module")
def host_lib():
    subprocess.check_call(["make", "-s", "-C", os.path.join(PKG, "csrc")])
    subprocess.check_call(["make", "-s", "-C", os.path.join(PKG, "host")])
    return os.path.join(PKG, "libloadflow_b200.so")


@pytest.fixture(scope="module")
def ref_lib():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])
    return os.path.join(ROOT, "oracle", "_ref", "libloadflow_ref.a")


@pytest.mark.parametrize("suite", SUITES)
def test_shim_is_faithful_on_reference_library(ref_lib, suite):
    """The same suites pass against the reference library itself (built from
    /root/reference/proj/src by oracle/ref.mk): the shim hides no failures and
    the suites pin behaviour the reference really has."""
    os.makedirs(BUILD, exist_ok=True)
    src = os.path.join(REF_TESTS, f"test_{suite}.cpp")
    exe = os.path.join(BUILD, f"ref_test_{suite}")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(ref_lib):
        subprocess.check_call([
            "g++", "-std=c++20", "-O1", "-w", "-include", "cstdint",
            "-I", os.path.join(ROOT, "tests", "conformance"),
            "-I", "/root/reference/proj/include",
            src, "-o", exe, ref_lib, "-lpthread"])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "failed: 0" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes(host_lib, suite):
    os.makedirs(BUILD, exist_ok=True)
    src = os.path.join(REF_TESTS, f"test_{suite}.cpp")
    exe = os.path.join(BUILD, f"test_{suite}")
    if not os.path.exists(exe) or os.path.getmtime(exe) < max(
            os.path.getmtime(src), os.path.getmtime(host_lib)):
        subprocess.check_call([
            "g++", "-std=c++20", "-O1", "-w",
            "-I", os.path.join(ROOT, "tests", "conformance"),
            "-I", os.path.join(ROOT, "include"),
            src, "-o", exe, "-L", PKG, "-lloadflow_b200", f"-Wl,-rpath,{PKG}", "-lpthread"])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, f"reference suite test_{suite} failed:\n{r.stderr[-4000:]}"
    assert "failed: 0" in r.stdout
