"""Drop-in check: the reference's own doctest suites (schedule, profile,
costmodel, planner) compiled unmodified against include/pipesim/*.hpp and
linked with libp2bw.so (oracle/Makefile target `dropin`).  The binaries are
built here from /root/reference; the GPU suites (semantics, acceptance) run
in tests/test_engine_linear_gpu.py."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


@pytest.mark.skipif(not (BIN / "dropin_host_tests").exists(), reason="drop-in harness not built")
def test_reference_host_suites_pass_on_libp2bw():
    r = subprocess.run([str(BIN / "dropin_host_tests")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "failed: 0 | assertions:" in r.stdout


@pytest.mark.skipif(not (BIN / "ref_tests").exists(), reason="reference not built here")
def test_doctest_shim_runs_reference_suites_on_reference():
    r = subprocess.run([str(BIN / "ref_tests")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
