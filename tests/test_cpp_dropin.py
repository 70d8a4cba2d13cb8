"""Drop-in proof: the REFERENCE's own unit tests (proj/tests/test_pipeline.cpp,
test_binning.cpp, test_csr.cpp, test_bench.cpp -- the last runs the reference's bench.cpp
run_benchmark over this library), compiled unmodified and in place against this repo's
C++ headers (include/spgemm/*.hpp) and libspgemm_b200.so by tests/cpp/Makefile.
The binaries are built in the build container (where /root/reference exists) and
travel with the repo snapshot; the tests skip when they are absent."""
import os
import subprocess

import pytest

BUILD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build")


def _run(name):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (make -C tests/cpp needs /root/reference)")
    res = subprocess.run([path], capture_output=True, text=True, timeout=900)
    failed = [l for l in res.stdout.splitlines() if l.startswith("[FAIL]") or "FAILED" in l]
    return res, failed


def test_reference_test_csr_host():
    res, failed = _run("test_csr")
    assert res.returncode == 0 and not failed, res.stdout[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_pipeline", "test_binning", "test_bench"])
def test_reference_unit_tests_on_b200(name):
    res, failed = _run(name)
    assert res.returncode == 0 and not failed, res.stdout[-4000:]
    assert "0 failed" in res.stdout
