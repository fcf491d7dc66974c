"""Parity at the BENCHMARKED shapes ("Next round" item 1).

The headline bench runs cfg3 (ChainMlp 16 x 4096 + scalar head, k = 8
workers x B_w = 128 rows = M 1024) and cfg4 (ResNet18-width ConvNet on 32 x 32
images). The GEMM plans those shapes select -- the CTA-pair forward with the
240-wide tiles (whose 18th column tile is 16 wide), the 192-wide pair wgrad at
K = 1024 contributor rows, the split-K dgrad at M = 128 and the pair split-K
dgrad at M = 256 / 384 / 512 -- only run at these sizes, so they are checked
here against CPU checkers on the same inputs:

* cfg3 widths at reduced depth (4096 x 4 + 1, k = 8, B_w = 128) against the
  UNMODIFIED reference (oracle/_ref, spb.cpp + model.cpp compiled from the
  reference's sources; one worker per thread);
* the full cfg3 depth (4096 x 16 + 1) against oracle/batched.py, the fp64
  BLAS restatement pinned to oracle/_ref in tests/test_oracle.py, including
  the bench's momentum 0.9 / weight decay 1e-4 optimizer and its default
  optimizer placement (fused into the <= 512-row wgrad epilogues);
* cfg4's ConvNet widths at 32 x 32 against oracle/conv_oracle.py.

Tolerances as everywhere (north_star): aggregated per-layer gradients 1e-5
relative, weights after N steps 1e-4 relative (norm-wise per layer). The
weight CHANGE W_N - W_0 is checked too, at 1e-4 of its norm plus the fp32
storage rounding of the weights (4 roundings of 2^-24 |w|): the updates of
the first layers are ~1e-4 of the weights, below fp32 resolution otherwise.
"""
import os

import numpy as np
import pytest

from conftest import rel_err
from oracle import batched
from oracle.oracle import fp32_round

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-5
WEIGHT_TOL = 1e-4


def delta_ok(got, w0, want) -> bool:
    """||(got - w0) - (want - w0)|| within 1e-4 of ||want - w0|| plus fp32 storage rounding."""
    d = np.asarray(got, np.float64) - w0
    dw = want - w0
    return np.linalg.norm(d - dw) <= 1e-4 * np.linalg.norm(dw) + 4 * 2.0**-24 * np.linalg.norm(want)


def _rows(orc, seed, s, k, bw, N):
    return np.concatenate([orc.draw_batch(seed, s, j, bw, N) for j in range(1, k + 1)])


def test_cfg3_width_step_matches_reference(orc, ref):
    """4096-wide layers, k = 8, B_w = 128 (the headline GEMM shapes at
    M = 1024 rows) against the compiled reference: the step-1 aggregate of
    every layer, and the weights after one step on the default (fused)
    optimizer placement."""
    from oracle.oracle import RefModel
    from paper_2111_10672_b200 import spb

    widths, k, bw, N, seed = [4096] * 4 + [1], 8, 128, 2048, 11
    X, Y, W = spb.gen_chain_mlp(widths, N, 7)
    W64 = [b.astype(np.float64) for b in W]
    m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw)
    try:
        m.set_optimizer(0.0)
        m.set_fused_update(0)
        m.train_steps(seed, 1, 1)
        grads = m.get_grads()
        assert np.array_equal(m.last_batch(k * bw), _rows(orc, seed, 1, k, bw, N))
        m.set_params(W)
        m.set_optimizer(0.01)
        m.set_fused_update(2)
        m.train_steps(seed, 1, 1)
        after = m.get_params()
    finally:
        m.close()
    r = RefModel(ref, widths, X.astype(np.float64), Y.astype(np.float64), W64)
    r.step(k, k * bw, 1.0, seed, 1, False, min(8, os.cpu_count() or 1))
    g_ref = [a - b for a, b in zip(W64, r.get_params())]
    for l, (a, b) in enumerate(zip(grads, g_ref)):
        assert rel_err(a, b) <= GRAD_TOL, (l, rel_err(a, b))
    for l, (a, b, w0) in enumerate(zip(after, g_ref, W64)):
        want = w0 - 0.01 * b  # x -= lr g (spb.cpp:196)
        assert rel_err(a, want) <= WEIGHT_TOL
        assert delta_ok(a, w0, want), l


@pytest.mark.parametrize("full", [False, True])
def test_cfg3_full_depth_matches_batched_oracle(orc, full):
    """The exact bench workload (cfg3: 4096 x 16 + 1, k = 8, B_w = 128,
    N = 8192, data seed 7, step seed 11, lr 0.01, momentum 0.9, wd 1e-4):
    step-1 aggregate (unfused, every layer) and the weights after 3 steps on
    the default optimizer placement, SPB and full backprop."""
    from paper_2111_10672_b200 import spb

    widths, k, bw, N, seed = [4096] * 16 + [1], 8, 128, 8192, 11
    lr, mu, wd = 0.01, 0.9, 1e-4
    X, Y, W = spb.gen_chain_mlp(widths, N, 7)
    m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw)
    try:
        m.set_optimizer(0.0)
        m.set_fused_update(0)
        m.train_steps(seed, 1, 1, full_backprop=full)
        grads = m.get_grads()
        m.set_params(W)
        m.set_optimizer(lr, mu, wd)
        m.set_fused_update(2)
        m.train_steps(seed, 1, 3, full_backprop=full)
        after = m.get_params()
    finally:
        m.close()
    X64, Y64 = X.astype(np.float64), Y.astype(np.float64)
    P = [b.astype(np.float64) for b in W]
    W0 = [p.copy() for p in P]
    bufs = [np.zeros_like(p) for p in P]
    for s in range(1, 4):
        rows = _rows(orc, seed, s, k, bw, N)
        g = batched.aggregate_step(widths, X64[rows], Y64[rows], P, k, bw, full)
        if s == 1:
            for l, (a, b) in enumerate(zip(grads, g)):
                assert rel_err(a, b) <= GRAD_TOL, (l, rel_err(a, b))
        batched.sgd_update(P, g, lr, mu, wd, bufs)
    for l, (a, b, w0) in enumerate(zip(after, P, W0)):
        assert rel_err(a, b) <= WEIGHT_TOL
        assert delta_ok(a, w0, b), (l, rel_err(a.astype(np.float64) - w0, b - w0))


def test_cfg4_resnet18_widths_match_conv_oracle(orc):
    """cfg4's ConvNet (32 x 32 x 3, 3 x 3 convs 64,64,128/2,128,256/2,256,
    512/2,512, pool, head 10) at k = 8, B_w = 16: the step-1 aggregate and
    the weights after 3 plain-SGD steps against the fp64 conv oracle."""
    from oracle.conv_oracle import ConvOracle
    from paper_2111_10672_b200 import spb

    shape, convs, nout = (32, 32, 3), [(64, 1), (64, 1), (128, 2), (128, 1), (256, 2), (256, 1), (512, 2), (512, 1)], 10
    k, bw, N, seed, lr = 8, 16, 512, 11, 0.01
    X, Y, W = spb.gen_convnet(shape, convs, nout, N, 7)
    m = spb.ConvNet(shape, convs, nout, X, Y, W, k=k, per_worker_batch=bw)
    try:
        m.set_optimizer(0.0)
        m.set_fused_update(0)
        m.train_steps(seed, 1, 1)
        grads = m.get_grads()
        m.set_params(W)
        m.set_optimizer(lr)
        m.set_fused_update(2)
        m.train_steps(seed, 1, 3)
        after = m.get_params()
    finally:
        m.close()
    o = ConvOracle(shape, convs, nout)
    X64, Y64 = X.astype(np.float64), Y.astype(np.float64)
    B = [w.astype(np.float64) for w in W]
    W0 = [b.copy() for b in B]
    G = [b.copy() for b in B]
    o.spb_step(G, X64, Y64, k, bw, 1.0, seed, 1, orc)
    for l in range(o.L):
        assert rel_err(grads[l], W0[l] - G[l]) <= GRAD_TOL, (l, rel_err(grads[l], W0[l] - G[l]))
    for s in range(1, 4):
        o.spb_step(B, X64, Y64, k, bw, lr, seed, s, orc)
    for l in range(o.L):
        assert rel_err(after[l], B[l]) <= WEIGHT_TOL
        assert delta_ok(after[l], W0[l], B[l]), l


@pytest.mark.parametrize("width", [1024, 2048, 8192])
def test_cfg5_widths_match_batched_oracle(orc, width):
    """cfg5 (BASELINE configs[4]: the width sweep 1k-8k, k = 8, B_w = 128) at
    depth 4: the step-1 aggregate of every layer against oracle/batched.py
    (1e-5), SPB, on the GEMM plans those widths select."""
    from paper_2111_10672_b200 import spb

    widths, k, bw, N, seed = [width] * 4 + [1], 8, 128, 2048, 11
    X, Y, W = spb.gen_chain_mlp(widths, N, 7)
    m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw)
    try:
        m.set_optimizer(0.0)
        m.set_fused_update(0)
        m.train_steps(seed, 1, 1)
        grads = m.get_grads()
    finally:
        m.close()
    rows = _rows(orc, seed, 1, k, bw, N)
    g = batched.aggregate_step(widths, X[rows].astype(np.float64), Y[rows].astype(np.float64),
                               [b.astype(np.float64) for b in W], k, bw)
    for l, (a, b) in enumerate(zip(grads, g)):
        assert rel_err(a, b) <= GRAD_TOL, (width, l, rel_err(a, b))
