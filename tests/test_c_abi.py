"""The C-ABI from a plain C program (tests/c/abi_smoke.c): host entry points
on the CPU, a small device pipeline with cudaMalloc'ed buffers on the GPU --
no Python, ctypes or torch between the caller and libcvz_b200.so."""

import os
import subprocess

import pytest

from conftest import ROOT, has_gpu
from paper_2108_00529_b200 import _native

SRC = os.path.join(ROOT, "tests", "c", "abi_smoke.c")
LIBDIR = os.path.dirname(_native.LIB_PATH)
CUDA = "/usr/local/cuda"


def _build(tmp_path, cuda):
    exe = str(tmp_path / ("abi_smoke_gpu" if cuda else "abi_smoke"))
    cmd = ["gcc", "-O1", "-std=c11", SRC, "-I", os.path.join(ROOT, "include"), "-L", LIBDIR,
           "-lcvz_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    if cuda:
        cmd[1:1] = ["-DWITH_CUDA", "-I", f"{CUDA}/include"]
        cmd += ["-L", f"{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_client_host_entry_points(tmp_path):
    _native.load()  # builds are made by __graft_entry__.build(); fail loudly if missing
    r = subprocess.run([_build(tmp_path, cuda=False)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "c-abi smoke ok" in r.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_c_client_device_pipeline(tmp_path):
    r = subprocess.run([_build(tmp_path, cuda=True), "--gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "c-abi smoke ok" in r.stdout
