"""ConvNet SPB step (BASELINE configs[3]).

The reference has no convolutional model, so parity is UNPINNED against it:
the fp64 numpy oracle (oracle/conv_oracle.py) is pinned by finite
differences here, and the SPB rules it applies (suffix cutoffs, contributor
averaging, batch draws) are the reference-pinned ones (oracle.Oracle).
GPU tolerances are the ChainMlp ones: gradients 1e-5, weights after N steps
1e-4, relative.
"""
import numpy as np
import pytest

from oracle.conv_oracle import ConvOracle, col2im, im2col

SHAPE, CONVS, NOUT = (8, 8, 3), [(8, 1), (12, 2), (16, 1), (16, 2)], 3
N, K, BW, LR, SEED, DSEED = 64, 4, 4, 0.05, 5, 9


# "tall": 16 x 16 images, so the layer-1 wgrad GEMM has K = 16 samples x 256
# pixel rows = 4096 against a single 8 x 36 output tile -> the split-K path.
# "tma": 32 / 64-channel inputs -> implicit GEMM through TMA im2col maps
# (forward A operand and wgrad B operand), strides 1 and 2; "tma_tall": the
# im2col-B wgrad with K = 4096 pixel rows -> split-K.
CASES = {"small": (SHAPE, CONVS, NOUT), "tall": ((16, 16, 4), [(8, 1), (8, 2), (12, 1)], 2),
         "tma": ((8, 8, 3), [(32, 1), (32, 2), (64, 1), (32, 2)], 3),
         "tma_tall": ((16, 16, 3), [(32, 1), (32, 1), (64, 2)], 2)}


def _data():
    from paper_2111_10672_b200 import spb

    return spb.gen_convnet(SHAPE, CONVS, NOUT, N, DSEED)


@pytest.mark.parametrize("shape,convs", [((6, 6, 3), [(4, 1), (5, 2), (6, 1)]), ((5, 7, 2), [(3, 2), (4, 2)])])
def test_conv_oracle_matches_finite_differences(shape, convs):
    from paper_2111_10672_b200 import spb

    X, Y, W = spb.gen_convnet(shape, convs, 2, 6, 1)
    o = ConvOracle(shape, convs, 2)
    B = [w.astype(np.float64) for w in W]
    g = o.partial_gradient(B, X, Y, o.L)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for l in range(o.L):
        for _ in range(6):
            i = int(rng.integers(len(B[l])))
            bp = [b.copy() for b in B]
            bm = [b.copy() for b in B]
            bp[l][i] += eps
            bm[l][i] -= eps
            fd = (o.loss(bp, X, Y) - o.loss(bm, X, Y)) / (2 * eps)
            assert abs(fd - g[l][i]) <= 1e-5 * max(1e-3, abs(fd))


def test_col2im_is_im2col_adjoint():
    rng = np.random.default_rng(3)
    for stride in (1, 2):
        x = rng.standard_normal((2, 5, 6, 3))
        cols, _ = im2col(x, stride)
        d = rng.standard_normal(cols.shape)
        assert np.isclose((cols * d).sum(), (x * col2im(d, x.shape, stride)).sum())


def test_partial_gradient_suffix_blocks():
    """Covered blocks of a partial pass equal the full pass's (test_spb.cpp:101-116 for this model)."""
    X, Y, W = _data()
    o = ConvOracle(SHAPE, CONVS, NOUT)
    B = [w.astype(np.float64) for w in W]
    full = o.partial_gradient(B, X[:8], Y[:8], o.L)
    for s in range(1, o.L + 1):
        part = o.partial_gradient(B, X[:8], Y[:8], s)
        for l in range(o.L):
            if l >= o.L - s:
                assert np.allclose(part[l], full[l], rtol=0, atol=0)
            else:
                assert part[l] is None


def test_block_dims():
    from paper_2111_10672_b200 import spb

    assert spb.convnet_block_dims((32, 32, 3), [(64, 1), (128, 2)], 10) == [64 * 27 + 64, 128 * 576 + 128, 10 * 128 + 10]


def _rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["small", "tma"])
def test_conv_loss_and_partial_backprop_match_oracle(case):
    from paper_2111_10672_b200 import spb

    shape, convs, nout = CASES[case]
    X, Y, W = spb.gen_convnet(shape, convs, nout, N, DSEED)
    o = ConvOracle(shape, convs, nout)
    B = [w.astype(np.float64) for w in W]
    m = spb.ConvNet(shape, convs, nout, X, Y, W, k=K, per_worker_batch=BW)
    try:
        assert m.loss() == pytest.approx(o.loss(B, X, Y), rel=1e-5)
        batch = np.array([3, 17, 5, 60, 41, 8, 8, 22], dtype=np.int32)
        for s in range(1, o.L + 1):
            pg = spb.partial_backprop(m, None, batch, s)
            want = o.partial_gradient(B, X[batch], Y[batch], s)
            assert pg.covered_from == o.L - s + 1
            for l in range(o.L):
                if want[l] is None:
                    continue
                assert _rel(pg.blocks[l], want[l]) <= 1e-5, (s, l)
    finally:
        m.close()


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["small", "tall", "tma", "tma_tall"])
@pytest.mark.parametrize("full", [False, True])
def test_conv_spb_steps_match_oracle(orc, full, case):
    from paper_2111_10672_b200 import spb

    shape, convs, nout = CASES[case]
    X, Y, W = spb.gen_convnet(shape, convs, nout, N, DSEED)
    o = ConvOracle(shape, convs, nout)
    B = [w.astype(np.float64) for w in W]
    m = spb.ConvNet(shape, convs, nout, X, Y, W, k=K, per_worker_batch=BW)
    try:
        m.set_optimizer(LR)
        m.train_steps(SEED, 1, 3, full_backprop=full)
        got = m.get_params()
        idx = m.last_batch(K * BW)
    finally:
        m.close()
    want_idx = np.concatenate([orc.draw_batch(SEED, 3, j, BW, N) for j in range(1, K + 1)])
    assert np.array_equal(idx, want_idx)
    for s in range(1, 4):
        o.spb_step(B, X.astype(np.float64), Y.astype(np.float64), K, BW, LR, SEED, s, orc, full=full)
    for l in range(o.L):
        assert _rel(got[l], B[l]) <= 1e-4, l


@pytest.mark.gpu
def test_conv_step_host_matches_device_draw(orc):
    """spb_step_host (host images in) = the device-drawn step on the same rows."""
    from paper_2111_10672_b200 import spb

    X, Y, W = _data()
    rows = np.concatenate([orc.draw_batch(SEED, 1, j, BW, N) for j in range(1, K + 1)])
    a = spb.ConvNet(SHAPE, CONVS, NOUT, X, Y, W, k=K, per_worker_batch=BW)
    b = spb.ConvNet(SHAPE, CONVS, NOUT, X, Y, W, k=K, per_worker_batch=BW)
    try:
        a.set_optimizer(LR)
        b.set_optimizer(LR)
        a.train_steps(SEED, 1, 1)
        b.step_host(np.ascontiguousarray(X[rows]), np.ascontiguousarray(Y[rows]))
        for pa, pb in zip(a.get_params(), b.get_params()):
            assert np.array_equal(pa, pb)
    finally:
        a.close()
        b.close()
