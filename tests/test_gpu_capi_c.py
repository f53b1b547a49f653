"""The C ABI from plain C: examples/capi_demo.c built with gcc against libgrkan_b200.so and run.

No Python or torch on the data path -- what a cgo / JNI / C++ binding of the
reference's forward_tensor / backward_blocked would do.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_through_the_c_abi(tmp_path):
    lib = os.path.join(ROOT, "paper_2505_13813_b200", "_lib")
    orc = os.path.join(ROOT, "oracle", "_build")
    if not os.path.exists(os.path.join(orc, "liboracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    exe = str(tmp_path / "capi_demo")
    cuda = "/usr/local/cuda"
    subprocess.run(["gcc", "-O2", "-std=c11", os.path.join(ROOT, "examples", "capi_demo.c"), "-o", exe,
                    "-I", os.path.join(ROOT, "include"), "-I", cuda + "/include",
                    "-L", lib, "-lgrkan_b200", "-L", orc, "-loracle", "-L", cuda + "/lib64", "-lcudart", "-lm",
                    "-Wl,-rpath," + lib + ":" + orc + ":" + cuda + "/lib64"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "capi demo ok" in out.stdout and "bitwise" in out.stdout
