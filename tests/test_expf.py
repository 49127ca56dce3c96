"""The device/host glibc expf port (paper_2602_12675_b200/csrc/expf_glibc.cuh) against this
host's libm expf on ALL 2^32 float inputs (CPU; compiled from the same header by
tests/cpp/expf_check.cpp). The router's bit-exact mask depends on it."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def test_expf_port_matches_libm_exhaustively(tmp_path):
    exe = tmp_path / "expf_check"
    src = os.path.join(HERE, "cpp", "expf_check.cpp")
    inc = os.path.join(os.path.dirname(HERE), "paper_2602_12675_b200", "csrc")
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-pthread", "-I", inc, "-o", str(exe), src],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches 0" in r.stdout, r.stdout
