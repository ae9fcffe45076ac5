"""The C ABI from plain C (examples/crd_example.c, no Python): it compiles and links against
include/mvn.h + libmvn.so; without a GPU it must fail loudly with MVN_E_CUDA (no CPU fallback);
on a B200 it runs end to end (mvn_crd), and its log P_k and regions equal the oracle's on the
inputs the C program generated (north_star bars: |dlog P_k| <= 1e-8, identical order and k*)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "crd_example")


def build_example():
    import paper_2405_14892_b200 as mvn
    mvn.lib()                                            # libmvn.so present (built by build())
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "crd_example.c"), "-L", os.path.join(ROOT, "paper_2405_14892_b200"),
           "-lmvn", "-Wl,-rpath," + os.path.join(ROOT, "paper_2405_14892_b200"), "-lm", "-o", EXE]
    subprocess.check_call(cmd)


def test_c_example_builds_and_fails_loudly_without_gpu():
    import torch
    build_example()
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by test_c_example_runs_on_gpu")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert r.returncode == 4, (r.returncode, r.stdout, r.stderr)      # MVN_E_CUDA
    assert "mvn_create" in r.stderr


@pytest.mark.gpu
def test_c_example_runs_on_gpu(cuda_device, tmp_path):
    import numpy as np
    import oracle
    build_example()
    dump = str(tmp_path / "crd.bin")
    r = subprocess.run([EXE, "20", "2000", "4", dump], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "region for 1-alpha = 0.95" in r.stdout and "sm_100a" in r.stdout
    raw = open(dump, "rb").read()
    n = int(np.frombuffer(raw[:8], dtype=np.int64)[0])
    off = 8
    def take(dt, cnt):
        nonlocal off
        a = np.frombuffer(raw[off:off + 8 * cnt], dtype=dt)
        off += 8 * cnt
        return a
    xy = take(np.float64, 2 * n).reshape(n, 2)
    mu = take(np.float64, n)
    order = take(np.int64, n)
    logP = take(np.float64, n)
    kstar = take(np.int64, 4)
    conf = [0.80, 0.90, 0.95, 0.99]
    ref = oracle.crd(xy, mu, 1.0, 0.1, 0.5, 1e-8, 0.0, 2000, 4, 3001, conf, chunk=500, nthreads=8)
    assert np.array_equal(order, ref.order)
    assert np.max(np.abs(logP - ref.logp)) <= 1e-8
    assert np.array_equal(kstar, ref.k_star)
