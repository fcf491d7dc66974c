"""Native (C/C++/CUDA) test programs: the GEMM numerics probe (the C++ drop-in
for the reference API is tests/test_dropin.py). Compiling needs no GPU (CPU
tests); running does (gpu tests)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

BUILD = os.path.join(ROOT, "build")
NVCC = "/usr/local/cuda/bin/nvcc"


def _build_probe():
    os.makedirs(BUILD, exist_ok=True)
    out = os.path.join(BUILD, "gemm_probe")
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-I",
                    os.path.join(ROOT, "include"), "-o", out, os.path.join(ROOT, "tests/native/gemm_probe.cu"),
                    os.path.join(ROOT, "paper_2111_10672_b200/csrc/gemm.cu")], check=True, capture_output=True)
    return out


def test_gemm_probe_compiles():
    assert os.path.exists(_build_probe())


@pytest.mark.gpu
def test_gemm_probe_numerics():
    r = subprocess.run([_build_probe()], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "GEMM PROBE OK" in r.stdout


@pytest.mark.gpu
def test_gemm_probe_benchmark_shapes():
    """The exact cfg3 GEMM shapes / layouts / epilogues with the planner's own
    choices (pair 240 forward, pair 192 wgrad at K = 1024, split-K dgrads,
    the fused-optimizer wgrad at K <= 512) against fp64."""
    r = subprocess.run([_build_probe(), "shapes"], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "GEMM SHAPES OK" in r.stdout
    # the plans the 1-GPU cfg3 step ships (profiles/r01_launches_cfg3_summary_v2.json)
    assert re.search(r"shape forward \(tanh epilogue\)\s+M=1024 N=4096 K=4096 plan=2sm/pn240/sp1", r.stdout)
    assert re.search(r"shape wgrad \(alpha epilogue\)\s+M=4096 N=4096 K=1024 plan=2sm/pn192/sp1", r.stdout)
    # the same shapes with the 1-CTA kernels' column-sum bias warps (SPB_BIAS=colsum)
    r = subprocess.run([_build_probe(), "shapes"], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, SPB_BIAS="colsum"))
    assert r.returncode == 0 and "GEMM SHAPES OK" in r.stdout, r.stdout + r.stderr
