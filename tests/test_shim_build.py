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


REF_INC = "/root/reference/proj/include"


def test_dropin_compiles_beside_reference_headers(tmp_path):
    """The drop-in header builds ON the reference's own types: one translation unit includes
    sla2_b200/sla2.hpp and then the reference's tape.hpp / model.hpp / training.hpp (the callers
    of the hot path) -- no redefinition, the specializations precede every use."""
    import pytest
    if not os.path.isdir(REF_INC):
        pytest.skip("reference headers absent (GPU box)")
    src = tmp_path / "tu.cpp"
    src.write_text('#include "sla2_b200/sla2.hpp"\n#ifndef SLA2_B200_MODE_REFERENCE\n#error wrong mode\n#endif\n'
                   '#include "sla2/tape.hpp"\n#include "sla2/model.hpp"\n#include "sla2/training.hpp"\n'
                   'int main() { return 0; }\n')
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include", str(src)], check=True)
