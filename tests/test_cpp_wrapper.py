"""The C++ drop-in header (gs::freq2wave / apply_* / solve_least_squares over
the C-ABI) compiles and links against libgs_b200.so on CPU; on a GPU the demo
program (reference-test-shaped checks) runs and exits 0."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "wrapper_demo.cpp")
LIBDIR = os.path.join(ROOT, "paper_1607_04091_b200")


def build(tmp_path):
    exe = os.path.join(str(tmp_path), "wrapper_demo")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-o", exe, SRC,
                           f"-I{os.path.join(ROOT, 'tests', 'cpp', 'shim')}", f"-I{os.path.join(LIBDIR, 'cpp')}",
                           f"-I{os.path.join(LIBDIR, 'cpp', 'include')}", f"-I{os.path.join(ROOT, 'include')}",
                           f"-L{LIBDIR}", "-lgs_b200", f"-Wl,-rpath,{LIBDIR}"])
    return exe


def test_wrapper_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_wrapper_runs_on_gpu(tmp_path):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, (out.returncode, out.stdout, out.stderr)
    assert "wrapper ok" in out.stdout
