"""The shared-reciprocal division (physics.cuh rcp_div / div_by) is bitwise
the device's own IEEE a / b: built here from tests/cuda/div_check.cu and run
over ~10^9 operand pairs per mode (random bit patterns of every class,
normal operands, near-tie quotients)."""
import ctypes as C
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "paper_1704_01144_b200", "csrc")


@pytest.fixture(scope="module")
def divlib(tmp_path_factory, gpu):
    out = str(tmp_path_factory.mktemp("div") / "libdivcheck.so")
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                    "--fmad=false", "-Xcompiler", "-fPIC", "-shared", "-I", CSRC, "-o", out,
                    os.path.join(HERE, "cuda", "div_check.cu")], check=True)
    lib = C.CDLL(out)
    lib.div_check.argtypes = [C.c_ulonglong, C.c_ulonglong, C.c_int, C.POINTER(C.c_ulonglong)]
    return lib


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_shared_reciprocal_division_is_ieee(divlib, mode):
    bad = C.c_ulonglong(0)
    assert divlib.div_check(1 << 30, 12345 + mode, mode, C.byref(bad)) == 0
    assert bad.value == 0
