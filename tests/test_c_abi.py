"""The C ABI from plain C (tests/c/abi_closed_form.c): compiled with gcc against the in-tree
libtm_w4a16.so and libcudart only -- no Python binding, no torch -- so the boundary is usable
as a standalone library.  Compiling and linking runs here; the GPU test executes it."""

import os
import subprocess

import pytest

from paper_2508_15601_b200 import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "abi_closed_form.c")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _compile(tmp_path):
    lib = build.build()
    exe = str(tmp_path / "abi_closed_form")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
           SRC, "-o", exe, "-L", os.path.dirname(lib), "-ltm_w4a16", "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm",
           "-Wl,-rpath," + os.path.dirname(lib) + ":" + os.path.join(CUDA, "lib64")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_consumer_compiles_and_links(tmp_path):
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.gpu
def test_c_consumer_closed_form_and_error_paths(tmp_path):
    exe = _compile(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok:" in r.stdout
