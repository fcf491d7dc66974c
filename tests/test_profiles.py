"""B200 task profiles for the Jigsaw simulator.

The emitted CSV must parse and validate under the reference's own
ProfileTable::from_csv (profile.cpp:118-171) and interpolate through its
forward_time / backward_time / peak_memory / task_demand (profile.cpp:67-92),
exactly at the knots.
"""
import numpy as np
import pytest

from paper_2111_10672_b200 import jigsaw_profiles as jp


def _rows(model, L, batch, fwd, bwd, mem, grad):
    return [f"{model},{s / L:.6g},{fwd[s - 1]:.4f},{bwd[s - 1]:.4f},{mem[s - 1]:.4f},{grad:.3f},{batch}"
            for s in range(1, L + 1)]


def test_emitted_schema_parses_in_reference(ref):
    L = 16
    fwd = np.full(L, 1.25)
    bwd = np.cumsum(np.full(L, 0.1))
    mem = 2.0 + np.cumsum(np.full(L, 0.05))
    grad = jp.grad_size_mb([4096] * 16 + [1])
    csv = jp.to_csv(_rows("ChainMlp-16x4096", L, 128, fwd, bwd, mem, grad))
    assert csv.splitlines()[0] == jp.HEADER
    for s in range(1, L + 1):
        q = ref.profile_query(csv, "ChainMlp-16x4096", s / L)
        assert q["forward_ms"] == pytest.approx(fwd[s - 1], abs=1e-4)
        assert q["backward_ms"] == pytest.approx(bwd[s - 1], abs=1e-4)
        assert q["peak_mem_gb"] == pytest.approx(mem[s - 1], abs=1e-4)
        assert q["batch"] == 128
    # worker j of k = 8 (fraction j/8) lands on a knot for L = 16
    q = ref.profile_query(csv, "ChainMlp-16x4096", 3 / 8)
    assert q["duration_ms"] == pytest.approx(fwd[5] + bwd[5], abs=1e-3)
    assert q["comm_mb"] == pytest.approx(grad * 3 / 8, rel=1e-6)


def test_grad_size_matches_reference_table_units():
    # The reference table lists MiB of fp32 gradients (ResNet101: 44.5M params -> 170).
    assert jp.grad_size_mb([1024, 1024, 1]) == pytest.approx(4 * (1024 * 1024 + 1024 + 1024 + 1) / 2**20)


def test_reference_rejects_decreasing_backward(ref):
    from oracle.oracle import OracleError

    csv = jp.to_csv(["m,0.5,1.0,2.0,1.0,10.000,8", "m,1,1.0,1.5,1.0,10.000,8"])
    with pytest.raises(OracleError):
        ref.profile_query(csv, "m", 1.0)


@pytest.mark.gpu
def test_b200_profile_rows_are_valid(ref):
    widths = [64, 96, 80, 48, 1]
    rows = jp.measure("tiny", widths, 32, reps=3)
    assert len(rows) == len(widths) - 1
    csv = jp.to_csv(rows)
    prev_b, prev_m = -1.0, -1.0
    L = len(widths) - 1
    for s in range(1, L + 1):
        q = ref.profile_query(csv, "tiny", s / L)
        assert q["forward_ms"] > 0
        assert q["backward_ms"] >= prev_b and q["peak_mem_gb"] >= prev_m
        prev_b, prev_m = q["backward_ms"], q["peak_mem_gb"]
    assert prev_b > 0
