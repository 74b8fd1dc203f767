"""The C ABI is usable from plain C (no Python, no torch): examples/c_api_demo.c compiles and
links against libfls.so here; on a GPU it runs Algorithm 1 end to end (-u'' = pi^2 sin(pi x))."""
import os
import subprocess

import pytest

from paper_2602_10541_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(tmp_path):
    build()
    exe = str(tmp_path / "c_api_demo")
    lib = os.path.join(ROOT, "paper_2602_10541_b200")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-std=c11", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "c_api_demo.c"),
           "-L", lib, "-lfls", "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{lib}", "-Wl,-rpath,/usr/local/cuda/lib64", "-lm", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_compiles_and_links(tmp_path):
    _compile(tmp_path)


@pytest.mark.gpu
def test_c_demo_runs_algorithm_1(tmp_path):
    exe = _compile(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "relative L2 error" in r.stdout
