"""The C++ drop-in header (include/sla2_b200/sla2.hpp) compiles against the C ABI and links
(CPU); tests/test_gpu_shim.py runs the resulting binary on the GPU."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_shim_test(out):
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-o", out,
           "-L", os.path.join(ROOT, "paper_2602_12675_b200"), "-lsla2_b200",
           "-L", os.path.join(ROOT, "oracle"), "-l:liboracle.so",
           "-L", "/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2602_12675_b200") + ":" + os.path.join(ROOT, "oracle")
           + ":/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    return out


def test_shim_compiles_and_links(tmp_path):
    import oracle_ctypes  # noqa: F401  (builds liboracle.so when missing)
    oracle_ctypes.port()
    exe = build_shim_test(str(tmp_path / "test_shim"))
    assert os.path.exists(exe)
