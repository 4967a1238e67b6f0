"""The drop-in boundary from C: examples/capi_step.c runs one fused step
through include/mosaic_b200.h and libmosaic_b200.so with no Python or torch
(the way the reference's FFI would link it). CPU: it compiles and links
against the header and the library; GPU: it runs and checks itself (argmax vs
fp64 on sampled rows, exactly k commits)."""
import shutil
import subprocess

import pytest

from conftest import ROOT

CUDA = "/usr/local/cuda"


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc unavailable")
    lib_dir = ROOT / "paper_2601_06562_b200"
    exe = tmp_path / "capi_step"
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", str(ROOT / "examples" / "capi_step.c"),
           f"-I{ROOT / 'include'}", f"-I{CUDA}/include", f"-L{lib_dir}", "-lmosaic_b200", f"-L{CUDA}/lib64",
           "-lcudart", "-lm", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles_and_links(native_lib, tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_c_example_runs(native_lib, tmp_path):
    r = subprocess.run([str(_build(tmp_path))], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "capi ok" in r.stdout
