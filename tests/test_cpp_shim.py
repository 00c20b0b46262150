"""The C++ drop-in shim compiles like a reference caller, links libsk_b200.so, and
(on a GPU) reproduces the reference's identity-pair / rank-deficiency behaviour."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2605_28274_b200")


def compile_shim(tmp_path):
    exe = str(tmp_path / "shim_main")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp_shim_main.cpp"), "-L", LIBDIR, "-lsk_b200",
                           f"-Wl,-rpath,{LIBDIR}", "-o", exe])
    return exe


def test_shim_compiles_and_links(tmp_path):
    from paper_2605_28274_b200 import build
    build.build()
    assert os.path.exists(compile_shim(tmp_path))


@pytest.mark.gpu
def test_shim_runs_on_device(tmp_path):
    from paper_2605_28274_b200 import build
    build.build()
    r = subprocess.run([compile_shim(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "identity_pair=1 rank_deficient=1" in r.stdout
