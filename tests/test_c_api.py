"""The C ABI used from plain C (examples/c_api_demo.c): it compiles and links
against include/sketch_b200.h + libsketch_b200.so on CPU; on the GPU its
output equals the oracle (bucket hashes and the first SA row, bit-exact)."""

import os
import subprocess

import numpy as np
import pytest

from .conftest import ROOT

DEMO = os.path.join(ROOT, "examples", "c_api_demo.c")


def build_demo(tmp_path):
    exe = str(tmp_path / "c_api_demo")
    lib_dir = os.path.join(ROOT, "paper_1207_6365_b200")
    cmd = ["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", DEMO, "-o", exe,
           "-L", lib_dir, "-lsketch_b200", "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def test_c_demo_compiles_against_the_header(tmp_path):
    if not os.path.exists("/usr/local/cuda/include/cuda_runtime.h"):
        pytest.skip("CUDA headers not installed")
    assert os.path.exists(build_demo(tmp_path))


@pytest.mark.gpu
def test_c_demo_matches_oracle(tmp_path):
    from oracle import oracle as O

    out = subprocess.run([build_demo(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    lines = dict(line.split(" = ") for line in out.stdout.splitlines() if " = " in line)
    n, d, t = 1000, 4, 64
    h, s = O.hash_signs(n, t, 1)
    a = ((np.arange(n * d) % 7) - 3.0).reshape(n, d)
    sa = O.apply_dense(h, s, t, a)
    assert [int(x) for x in lines["bucket[0..3]"].split()] == h[:4].tolist()
    assert [float(x) for x in lines["SA[0][0..3] "].split()] == sa[0].tolist()


def test_c_mm_ingest_demo(tmp_path):
    """Matrix Market ingest from plain C (host only: runs without a GPU)."""
    if not os.path.exists("/usr/local/cuda/include/cuda_runtime.h"):
        pytest.skip("CUDA headers not installed")
    exe = str(tmp_path / "mm_demo")
    lib_dir = os.path.join(ROOT, "paper_1207_6365_b200")
    cmd = ["gcc", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "mm_ingest_demo.c"),
           "-o", exe, "-L", lib_dir, "-lsketch_b200", f"-Wl,-rpath,{lib_dir}"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    good = tmp_path / "s.mtx"
    good.write_text("%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 3\n1 1 2.5\n3 1 -1e-3\n2 2 4\n")
    out = subprocess.run([exe, str(good), "2"], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    lines = dict(line.split(" = ") for line in out.stdout.splitlines())
    assert lines["shape"] == "3 3" and lines["declared"] == "3" and lines["count"] == "4"
    assert lines["field symmetric"] == "0 1"
    assert lines["entry1"] == "2 0 -0.001"
    bad = tmp_path / "b.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 9 1.0\n")
    out = subprocess.run([exe, str(bad)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 1 and out.stdout.strip() == f"error = {bad}:3: index out of range"
