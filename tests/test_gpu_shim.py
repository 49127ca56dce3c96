"""Runs the reference's forward-path tests re-expressed against the C++ drop-in header."""
import subprocess

import pytest

from test_shim_build import build_shim_test

pytestmark = pytest.mark.gpu


def test_cpp_shim_against_oracle(cuda, tmp_path):
    import oracle_ctypes
    oracle_ctypes.port()
    exe = build_shim_test(str(tmp_path / "test_shim"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
