"""Parity of the B200 SPB path (through the C ABI) with the CPU oracle and the
reference's golden fixtures.

Tolerances (north_star, BASELINE.json): per-layer aggregated gradients within
1e-5 relative, weights after N steps within 1e-4 relative, both norm-wise per
layer (the reference's own FD check is norm-wise, verify.cpp:232-244), fp32
on the B200 against the fp64 reference fed the same fp32-rounded inputs.
Integer outputs (cutoffs, coverage, batch indices, op counts) are bit-exact.
"""
import numpy as np
import pytest

from conftest import load_golden, rel_err, unpack_blocks
from oracle.oracle import fp32_round
from paper_2111_10672_b200 import spb

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-5
WEIGHT_TOL = 1e-4


def make(widths, N, seed, k=1, bw=1):
    X, Y, W = spb.gen_chain_mlp(widths, N, seed)
    m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw)
    return m, X.astype(np.float64), Y.astype(np.float64), [b.astype(np.float64) for b in W]


SHAPES = [
    ([3, 4, 4, 4, 1], 24, 5),
    ([3, 5, 4, 1], 32, 1),
    ([37, 33, 20, 1], 100, 9),
    ([300, 257, 129, 1], 500, 3),
    ([784, 512, 512, 1], 1024, 7),
    ([64, 130, 96, 10], 200, 2),  # 10-wide head (throughput variant; oracle generalises 0.5||out-y||^2)
]


@pytest.mark.parametrize("widths,N,seed", SHAPES)
def test_partial_backprop_matches_oracle(orc, widths, N, seed):
    m, X, Y, W = make(widths, N, seed)
    if widths[-1] > 1:
        Y = np.repeat(Y[:, :1], widths[-1], axis=1)
    L = len(widths) - 1
    batch = np.random.default_rng(seed).integers(0, N, size=37).astype(np.int32)
    for suffix in range(1, L + 1):
        stats = spb.BackpropStats()
        pg = spb.partial_backprop(m, None, batch, suffix, stats)
        ops = np.zeros(L, dtype=np.int64)
        ref, cov = orc.partial_backprop(widths, X, Y, W, batch, suffix, ops)
        assert pg.covered_from == cov == L - suffix + 1
        assert stats.layer_ops == ops.tolist()
        for l in range(L):
            if ref[l] is None:
                assert pg.blocks[l].size == 0
            else:
                e = rel_err(pg.blocks[l], ref[l])
                assert e <= GRAD_TOL, (widths, suffix, l, e)


def test_suffix_blocks_bit_identical_to_full_pass():
    # test_spb.cpp:101-116 on the GPU: covered blocks are the same bits as the full pass.
    m, X, Y, W = make([64, 48, 40, 32, 1], 64, 4)
    batch = np.arange(0, 60, 3, dtype=np.int32)
    L = 4
    full = spb.partial_backprop(m, None, batch, L)
    for suffix in range(1, L + 1):
        part = spb.partial_backprop(m, None, batch, suffix)
        for l in range(L):
            if l + 1 >= part.covered_from:
                assert np.array_equal(part.blocks[l], full.blocks[l])
            else:
                assert part.blocks[l].size == 0


def test_partial_backprop_argument_errors():
    m, *_ = make([3, 4, 4, 4, 1], 24, 5)
    with pytest.raises(spb.ArgumentError):
        spb.partial_backprop(m, None, [0, 1], 0)
    with pytest.raises(spb.ArgumentError):
        spb.partial_backprop(m, None, [0, 1], 5)
    with pytest.raises(spb.ArgumentError):
        spb.partial_backprop(m, None, [], 1)
    with pytest.raises(spb.ArgumentError):
        spb.partial_backprop(m, None, [24], 1)


def test_golden_g1_partial_backprop():
    g = load_golden("g1_partial_backprop.npz")
    widths = g["widths"].tolist()
    m, *_ = make(widths, int(g["samples"]), int(g["seed"]))
    L = len(widths) - 1
    for suffix in range(1, L + 1):
        st = spb.BackpropStats()
        pg = spb.partial_backprop(m, None, g["batch"], suffix, st)
        assert pg.covered_from == int(g[f"cov_{suffix}"])
        assert st.layer_ops == g[f"ops_{suffix}"].tolist()
        for l, p in enumerate(unpack_blocks(g, f"pb{suffix}", L)):
            if p is None:
                assert pg.blocks[l].size == 0
                continue
            idx, val, norm, size = p
            assert pg.blocks[l].size == size
            assert rel_err(pg.blocks[l][idx], val) <= GRAD_TOL
    assert abs(m.loss() - float(g["loss"])) <= 1e-6 * abs(float(g["loss"]))


def test_aggregate_matches_oracle_and_protocol(orc):
    rng = np.random.default_rng(77)
    k, L = 4, 11
    dims = [1 + int(rng.integers(0, 4)) for _ in range(L)]
    grads = []
    for j in range(1, k + 1):
        cov = L - spb.suffix_layers(j, k, L) + 1
        blocks = [rng.uniform(-1, 1, size=dims[l]).astype(np.float32) if l + 1 >= cov else np.zeros(0, np.float32)
                  for l in range(L)]
        grads.append(spb.PartialGradient(blocks, cov))
    agg = spb.aggregate(grads, k)
    ref = orc.aggregate([[b.astype(np.float64) if b.size else None for b in g.blocks] for g in grads],
                        [g.covered_from for g in grads], k)
    for a, b in zip(agg, ref):
        assert rel_err(a, b) <= 1e-6
    broken = [spb.PartialGradient(list(g.blocks), g.covered_from) for g in grads]
    broken[0].covered_from -= 1
    with pytest.raises(spb.ProtocolError):
        spb.aggregate(broken, k)
    missing = [spb.PartialGradient(list(g.blocks), g.covered_from) for g in grads]
    missing[1].blocks[L - 1] = np.zeros(0, np.float32)
    with pytest.raises(spb.ProtocolError):
        spb.aggregate(missing, k)
    with pytest.raises(spb.ArgumentError):
        spb.aggregate(grads[:3], k)


def test_aggregate_hand_example():
    k = L = 3
    grads = []
    for j in range(1, k + 1):
        cov = L - spb.suffix_layers(j, k, L) + 1
        grads.append(spb.PartialGradient([np.array([3.0 * j], np.float32) if l + 1 >= cov else np.zeros(0, np.float32)
                                          for l in range(L)], cov))
    grads[2].blocks[0] = np.array([-2.5], np.float32)
    agg = spb.aggregate(grads, k)
    assert agg[2][0] == pytest.approx(6.0)
    assert agg[0][0] == -2.5


@pytest.mark.parametrize("fused", [0, 1, 2])
@pytest.mark.parametrize("widths,N,k,bw", [([3, 5, 4, 1], 32, 3, 2), ([37, 33, 20, 1], 100, 4, 5),
                                          ([128, 96, 80, 64, 48, 1], 256, 8, 16), ([784, 512, 512, 1], 4096, 4, 128),
                                          ([300, 257, 129, 96, 1], 2048, 4, 192)])
def test_spb_step_batches_grads_and_weights(orc, widths, N, k, bw, fused):
    """One device SPB step: batch indices bit-exact, the aggregated gradient
    (unfused path) within 1e-5 of the oracle's aggregate, weights within 1e-4
    (optimizer placement 0 / 1 / 2; the 192-row case mixes fused and unfused
    layers under the default 2); then 5 steps."""
    m, X, Y, W = make(widths, N, 13, k=k, bw=bw)
    L = len(widths) - 1
    lr, seed = 0.05, 11
    m.set_optimizer(lr)
    m.set_fused_update(fused)
    m.train_steps(seed, 1, 1)
    got = m.last_batch(k * bw)
    grads, covs = [], []
    for j in range(1, k + 1):
        b = orc.draw_batch(seed, 1, j, bw, N)
        assert (got[(j - 1) * bw:j * bw] == b).all()
        g, c = orc.partial_backprop(widths, X, Y, W, b, orc.suffix_layers(j, k, L))
        grads.append(g)
        covs.append(c)
    agg = orc.aggregate(grads, covs, k)
    if not fused:
        for l, (a, b) in enumerate(zip(m.get_grads(), agg)):
            assert rel_err(a, b) <= GRAD_TOL, (l, rel_err(a, b))
    P = [b.copy() for b in W]
    orc.spb_step(widths, X, Y, P, k, k * bw, lr, seed, 1)
    for a, b in zip(m.get_params(), P):
        assert rel_err(a, b) <= WEIGHT_TOL
    m.train_steps(seed, 2, 4)
    for s in range(2, 6):
        orc.spb_step(widths, X, Y, P, k, k * bw, lr, seed, s)
    for a, b in zip(m.get_params(), P):
        assert rel_err(a, b) <= WEIGHT_TOL


def test_golden_g2_trajectory():
    g = load_golden("g2_sgd_trajectory.npz")
    widths = g["widths"].tolist()
    k, B = int(g["k"]), int(g["B"])
    m, *_ = make(widths, int(g["samples"]), int(g["seed"]), k=k, bw=B // k)
    m.set_optimizer(float(g["lr"]))
    L = len(widths) - 1
    for s in range(1, int(g["steps"]) + 1):
        m.train_steps(int(g["step_seed"]), s, 1)
        got = m.last_batch(B)
        for j in range(1, k + 1):
            assert (got[(j - 1) * (B // k):j * (B // k)] == g[f"batch_{s}_{j}"]).all()
        for x, p in zip(m.get_params(), unpack_blocks(g, f"x{s}", L)):
            idx, val, norm, size = p
            assert rel_err(x[idx], val) <= WEIGHT_TOL


def test_golden_g3_ragged_aggregate(orc):
    g = load_golden("g3_ragged_aggregate.npz")
    widths = g["widths"].tolist()
    k, bw = int(g["k"]), int(g["bw"])
    m, X, Y, W = make(widths, int(g["samples"]), int(g["seed"]), k=k, bw=bw)
    m.set_optimizer(0.0)
    m.set_fused_update(False)
    m.train_steps(int(g["step_seed"]), 1, 1)
    for gr, p in zip(m.get_grads(), unpack_blocks(g, "agg", len(widths) - 1)):
        idx, val, norm, size = p
        assert rel_err(gr[idx], val) <= GRAD_TOL
        assert abs(np.linalg.norm(gr) - norm) <= GRAD_TOL * norm


def test_golden_g4_cfg1():
    """cfg1 (784-512-512-1, k=4, B_w=128): the step-1 aggregate and the
    weights after 10 SPB-SGD steps against the reference's own numbers."""
    g = load_golden("g4_cfg1.npz")
    widths = g["widths"].tolist()
    k, bw = int(g["k"]), int(g["bw"])
    m, *_ = make(widths, int(g["samples"]), int(g["seed"]), k=k, bw=bw)
    m.set_optimizer(float(g["lr"]))
    L = len(widths) - 1
    m.set_fused_update(False)  # step 1 unfused (aggregate readable), steps 2..10 fused
    m.train_steps(int(g["step_seed"]), 1, 1)
    m.set_fused_update(True)
    for gr, p in zip(m.get_grads(), unpack_blocks(g, "agg", L)):
        idx, val, norm, size = p
        assert rel_err(gr[idx], val) <= GRAD_TOL
        assert abs(np.linalg.norm(gr) - norm) <= GRAD_TOL * norm
    m.train_steps(int(g["step_seed"]), 2, int(g["steps"]) - 1)
    for x, p in zip(m.get_params(), unpack_blocks(g, "x10", L)):
        idx, val, norm, size = p
        assert rel_err(x[idx], val) <= WEIGHT_TOL
        assert abs(np.linalg.norm(x) - norm) <= WEIGHT_TOL * norm
    assert abs(m.loss() - float(g["loss10"])) <= 1e-4 * float(g["loss10"])


def test_full_backprop_baseline_matches_oracle(orc):
    widths, N, k, bw = [37, 33, 20, 1], 100, 4, 5
    m, X, Y, W = make(widths, N, 21, k=k, bw=bw)
    m.set_optimizer(0.05)
    m.train_steps(11, 1, 3, full_backprop=True)
    P = [b.copy() for b in W]
    for s in range(1, 4):
        orc.spb_step(widths, X, Y, P, k, k * bw, 0.05, 11, s, full=True)
    for a, b in zip(m.get_params(), P):
        assert rel_err(a, b) <= WEIGHT_TOL


def test_k1_spb_equals_full_backprop_bitwise():
    # verify.cpp:274-301 on the GPU: with k=1 SPB is plain SGD.
    widths = [64, 48, 32, 1]
    a, *_ = make(widths, 128, 3, k=1, bw=16)
    b, *_ = make(widths, 128, 3, k=1, bw=16)
    a.set_optimizer(0.1)
    b.set_optimizer(0.1)
    a.train_steps(5, 1, 6)
    b.train_steps(5, 1, 6, full_backprop=True)
    for x, y in zip(a.get_params(), b.get_params()):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("fused", [0, 1, 2])
def test_momentum_weight_decay_restatement(orc, fused):
    """Momentum SGD + wd (parity unpinned by the reference):
    device update (separate kernel, or fused into the wgrad epilogue) vs the
    oracle's PyTorch-semantics restatement over 3 steps."""
    widths, N, k, bw = [37, 33, 20, 1], 100, 4, 5
    lr, mu, wd, seed = 0.05, 0.9, 1e-2, 11
    m, X, Y, W = make(widths, N, 17, k=k, bw=bw)
    m.set_optimizer(lr, mu, wd)
    m.set_fused_update(fused)
    L = len(widths) - 1
    P = [b.copy() for b in W]
    bufs = [np.zeros_like(b) for b in W]
    for s in range(1, 4):
        grads, covs = [], []
        for j in range(1, k + 1):
            g, c = orc.partial_backprop(widths, X, Y, P, orc.draw_batch(seed, s, j, bw, N), orc.suffix_layers(j, k, L))
            grads.append(g)
            covs.append(c)
        agg = orc.aggregate(grads, covs, k)
        for l in range(L):
            orc.sgd_momentum(P[l], agg[l], bufs[l], lr, mu, wd, s == 1)
        m.train_steps(seed, s, 1)
    for a, b in zip(m.get_params(), P):
        assert rel_err(a, b) <= WEIGHT_TOL


def test_step_host_rows_equal_device_gather():
    widths, N, k, bw = [64, 48, 32, 1], 256, 4, 8
    a, X, Y, W = make(widths, N, 8, k=k, bw=bw)
    b, *_ = make(widths, N, 8, k=k, bw=bw)
    a.set_optimizer(0.1)
    b.set_optimizer(0.1)
    seed = 9
    idx = np.concatenate([spb.draw_batch(seed, 1, j, bw, N) for j in range(1, k + 1)])
    loss_h = b.step_host(np.ascontiguousarray(X[idx], dtype=np.float32), np.ascontiguousarray(Y[idx], dtype=np.float32))
    la = a.train_steps(seed, 1, 1, losses=True)
    assert float(la[0]) == loss_h
    for x, y in zip(a.get_params(), b.get_params()):
        assert np.array_equal(x, y)


def test_loss_matches_oracle(orc):
    widths, N = [300, 257, 129, 1], 777
    m, X, Y, W = make(widths, N, 3, k=2, bw=64)
    assert abs(m.loss() - orc.loss(widths, X, Y, W)) <= 1e-6 * orc.loss(widths, X, Y, W)


def test_deep_wide_step_properties():
    """cfg3-shaped step (4096-wide, k=8; L=8 here) at a reduced batch: SPB's
    aggregate equals the contributor mean of per-worker partial backprops on
    the same device (linearity of the aggregate), and training decreases the loss."""
    widths = [4096] * 8 + [1]
    k, bw, N = 8, 16, 1024
    X, Y, W = spb.gen_chain_mlp(widths, N, 7)
    m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw)
    del X, Y, W
    L = len(widths) - 1
    m.set_optimizer(0.0)
    m.set_fused_update(False)
    m.train_steps(11, 1, 1)
    agg = m.get_grads()
    batches = m.last_batch(k * bw)
    pgs = [spb.partial_backprop(m, None, batches[(j - 1) * bw:j * bw], spb.suffix_layers(j, k, L))
           for j in range(1, k + 1)]
    ref = spb.aggregate(pgs, k)
    for a, b in zip(agg, ref):
        assert rel_err(a, b) <= 1e-5
    m.set_optimizer(0.01)
    m.set_fused_update(True)
    l0 = m.train_steps(11, 2, 1, losses=True)[0]
    ls = m.train_steps(11, 3, 20, losses=True)
    assert np.isfinite(ls).all()
    assert ls[-5:].mean() < l0


def test_aggregate_repeated_calls_are_exact():
    """Regression: spb_aggregate's staging buffer was zeroed on the legacy
    default stream, unordered with the copies on the context's stream, and
    lost a worker's block about once in 15 calls. 40 calls on random blocks
    must all equal the host mean over contributors (spb.cpp:97-103)."""
    widths = [96, 80, 64, 1]
    k = 4
    X, Y, W = spb.gen_chain_mlp(widths, 64, 3)
    m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=4)
    L = len(widths) - 1
    rng = np.random.default_rng(0)
    dims = spb.block_dims(widths)
    try:
        for _ in range(40):
            pgs = []
            for j in range(1, k + 1):
                s = spb.suffix_layers(j, k, L)
                blocks = [rng.standard_normal(d).astype(np.float32) if l >= L - s else np.zeros(0, np.float32)
                          for l, d in enumerate(dims)]
                pgs.append(spb.PartialGradient(blocks, L - s + 1))
            got = spb.aggregate(pgs, k)
            for l in range(L):
                contrib = [pg.blocks[l] for pg in pgs if pg.blocks[l].size]
                want = np.sum(np.stack(contrib).astype(np.float64), axis=0) / len(contrib)
                assert np.allclose(got[l], want, rtol=1e-6, atol=1e-7)
    finally:
        m.close()


@pytest.mark.parametrize("fused", [0, 2])
@pytest.mark.parametrize("full", [False, True])
def test_chained_graph_bitwise_equals_single_steps(fused, full):
    """spb_set_chain: up to 16 iterations captured in one graph, iteration
    t+1's forward of layer l gated only on W_l of iteration t. Same kernels,
    same data order: weights and per-step losses must be bit-identical to one
    graph per iteration, over 11 steps (chunks 8 + 3) with momentum + wd."""
    widths, N, k, bw = [96, 128, 80, 64, 1], 512, 4, 16
    ms = []
    for chain in (1, 8):
        m, *_ = make(widths, N, 4, k=k, bw=bw)
        m.set_optimizer(0.05, 0.9, 1e-3)
        m.set_fused_update(fused)
        m.set_chain(chain)
        ms.append((m, m.train_steps(13, 1, 11, full_backprop=full, losses=True)))
    (a, la), (b, lb) = ms
    assert np.array_equal(la, lb)
    for x, y in zip(a.get_params(), b.get_params()):
        assert np.array_equal(x, y)


def test_set_chain_rejects_bad_values():
    m, *_ = make([8, 8, 1], 16, 1, k=1, bw=4)
    for bad in (0, 17, -1):
        with pytest.raises(spb.ArgumentError):
            m.set_chain(bad)


def test_trace_steps_timeline_and_results():
    """spb_trace_steps replays a traced chained graph twice: every op gets a
    begin <= end stamp, and the parameters equal 2 * steps untraced steps."""
    widths, N, k, bw = [64, 96, 48, 1], 256, 4, 8
    a, *_ = make(widths, N, 6, k=k, bw=bw)
    b, *_ = make(widths, N, 6, k=k, bw=bw)
    for m in (a, b):
        m.set_optimizer(0.05, 0.9, 1e-3)
    tr = a.trace_steps(3, 1, 3)
    b.train_steps(3, 1, 6)
    assert len(tr["t0"]) > 10 and (tr["t1"] >= tr["t0"]).all()
    assert set(np.unique(tr["sub"])) == {0, 1, 2}
    assert (tr["cls"] == 0).sum() == 3 * (len(widths) - 2)  # forward GEMMs
    for x, y in zip(a.get_params(), b.get_params()):
        assert np.array_equal(x, y)


def test_step_host_async_equals_step_host():
    """spb_step_host_async (double-buffered staging, copy stream, no host
    sync) must produce the same losses and weights as spb_step_host."""
    widths, N, k, bw = [64, 48, 32, 1], 256, 4, 8
    a, X, Y, W = make(widths, N, 8, k=k, bw=bw)
    b, *_ = make(widths, N, 8, k=k, bw=bw)
    a.set_optimizer(0.1, 0.9, 1e-3)
    b.set_optimizer(0.1, 0.9, 1e-3)
    batches = []
    for s in range(1, 6):
        idx = np.concatenate([spb.draw_batch(4, s, j, bw, N) for j in range(1, k + 1)])
        batches.append((np.ascontiguousarray(X[idx], dtype=np.float32), np.ascontiguousarray(Y[idx], dtype=np.float32)))
    want = [b.step_host(x, y) for x, y in batches]
    got = np.zeros(len(batches), dtype=np.float32)
    for i, (x, y) in enumerate(batches):
        a.step_host_async(x, y, got[i:i + 1])
    a.synchronize()
    assert np.array_equal(got, np.array(want, dtype=np.float32))
    for x, y in zip(a.get_params(), b.get_params()):
        assert np.array_equal(x, y)


def test_step_host_rejects_bad_host_arrays():
    """the C side copies hosted_rows x n_0 / n_L floats straight
    from the pointers, so wrong dtypes, non-contiguous views and short batches
    are rejected before the call instead of reading garbage."""
    widths, N, k, bw = [64, 48, 32, 1], 256, 4, 8
    m, X, Y, W = make(widths, N, 8, k=k, bw=bw)
    x = np.ascontiguousarray(X[:k * bw], dtype=np.float32)
    y = np.ascontiguousarray(Y[:k * bw], dtype=np.float32)
    for bad_x, bad_y in ((x.astype(np.float64), y), (np.asfortranarray(x), y), (x[:-1], y), (x, y[:, :0]),
                         (np.ascontiguousarray(np.zeros((k * bw, 65), np.float32))[:, :64], y)):
        with pytest.raises(spb.ArgumentError):
            m.step_host(bad_x, bad_y)
        with pytest.raises(spb.ArgumentError):
            m.step_host_async(bad_x, bad_y, np.zeros(1, np.float32))
    m.step_host(x, y)
    m.close()


def test_k1_spb_equals_plain_sgd_bitwise_50_iterations():
    """verify.cpp:274-301 through the DEVICE step: with k = 1 the single worker
    backpropagates every layer, so 50 SPB-SGD iterations are bit-identical to
    50 plain SGD (full-backprop) iterations on the same draws."""
    widths = [64, 48, 32, 1]
    a, *_ = make(widths, 256, 3, k=1, bw=16)
    b, *_ = make(widths, 256, 3, k=1, bw=16)
    a.set_optimizer(1e-2)
    b.set_optimizer(1e-2)
    la = a.train_steps(5, 1, 50, losses=True)
    lb = b.train_steps(5, 1, 50, full_backprop=True, losses=True)
    assert np.array_equal(la, lb)
    for x, y in zip(a.get_params(), b.get_params()):
        assert np.array_equal(x, y)


def test_aggregation_unbiased_through_device_step():
    """verify.cpp:303-341 through the DEVICE step: the mean of many SPB
    aggregates (each from fresh worker draws, k = 4) converges to the full
    gradient -- every layer's deviation within 3 standard errors."""
    widths, N, k, bw, trials = [12, 10, 8, 6, 1], 96, 4, 2, 3000
    m, X, Y, W = make(widths, N, 9, k=k, bw=bw)
    L = len(widths) - 1
    full = spb.partial_backprop(m, None, np.arange(N, dtype=np.int32), L).blocks  # full_gradient
    m.set_optimizer(0.0)
    m.set_fused_update(0)
    est = []
    for t in range(1, trials + 1):
        m.train_steps(77, t, 1)
        est.append([g.astype(np.float64) for g in m.get_grads()])
    for l in range(L):
        e = np.stack([x[l] for x in est])
        mean = e.mean(axis=0)
        se = np.sqrt(((e - mean) ** 2).sum() / trials / (trials - 1))
        dev = np.linalg.norm(mean - full[l])
        assert dev <= 3.0 * se, (l, dev / se)
