"""Gradient-noise estimator on the GPU.

empirical_variance (spb.cpp:212-265) runs, per trial, the SPB estimate and
the full-backprop baseline on the trial's worker batches, and per chunk a
stream of single-sample gradients. The GPU version follows the same sampling
protocol sample for sample, so its estimates must equal the reference's up
to fp32 rounding of the gradients (tolerance 1e-4 relative).
"""
import numpy as np
import pytest

WIDTHS, N, K, B, TRIALS, SEED, DSEED = [12, 10, 9, 8, 6, 1], 64, 4, 8, 25, 3, 17


def _ref_model(ref):
    from oracle.oracle import RefModel
    from paper_2111_10672_b200 import spb

    X, Y, W = spb.gen_chain_mlp(WIDTHS, N, DSEED)
    return RefModel(ref, WIDTHS, X.astype(np.float64), Y.astype(np.float64), [w.astype(np.float64) for w in W]), (X, Y, W)


def test_reference_estimators_agree_at_k1(ref):
    """At k = 1 the reference's oracle reproduces empirical_variance exactly
    (oracle.hpp:57-60): pins the reference plumbing the GPU test relies on."""
    rm, _ = _ref_model(ref)
    a = rm.empirical_variance(1, 8, 10, SEED)
    b = rm.variance_oracle(1, 8, 10, SEED)
    assert a["spb"] == pytest.approx(b["spb"], rel=1e-12)
    assert np.allclose(a["p_hat"], b["p_hat"], rtol=1e-12)


def test_reference_rejects_bad_config(ref):
    from oracle.oracle import OracleError

    rm, _ = _ref_model(ref)
    with pytest.raises(OracleError):
        rm.empirical_variance(3, 8, 5, SEED)


@pytest.mark.gpu
def test_gpu_empirical_variance_matches_reference(ref):
    from paper_2111_10672_b200 import spb

    rm, (X, Y, W) = _ref_model(ref)
    want = rm.empirical_variance(K, B, TRIALS, SEED)
    m = spb.ChainMlp(WIDTHS, X, Y, W, k=K, per_worker_batch=B // K)
    try:
        got = spb.empirical_variance(m, spb.SpbConfig(k=K, B=B), None, TRIALS, SEED)
    finally:
        m.close()
    assert got.spb == pytest.approx(want["spb"], rel=1e-4)
    assert got.baseline == pytest.approx(want["baseline"], rel=1e-4)
    assert got.spb_se == pytest.approx(want["spb_se"], rel=1e-3)
    assert np.allclose(got.p_hat, want["p_hat"], rtol=1e-4)
    assert np.allclose(got.p_se, want["p_se"], rtol=1e-3)
    # SPB trades variance for compute: never below the baseline's on average here.
    assert got.spb > got.baseline


@pytest.mark.gpu
def test_gpu_empirical_variance_argument_errors():
    from paper_2111_10672_b200 import spb

    X, Y, W = spb.gen_chain_mlp(WIDTHS, N, DSEED)
    m = spb.ChainMlp(WIDTHS, X, Y, W, k=K, per_worker_batch=B // K)
    try:
        with pytest.raises(spb.ArgumentError):
            spb.empirical_variance(m, spb.SpbConfig(k=K, B=2 * B), None, 5, SEED)
        with pytest.raises(spb.ArgumentError):
            spb.empirical_variance(m, spb.SpbConfig(k=K, B=B), None, 0, SEED)
    finally:
        m.close()
