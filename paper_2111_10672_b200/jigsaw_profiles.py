"""B200 task profiles for the Jigsaw simulator.

The reference schedules SPB worker tasks from a measured profile table
(jigsaw/cost/profile.hpp:20-80, data/profiles.csv): one row per knot
`model,fraction,forward_ms,backward_ms,peak_mem_gb,grad_size_mb,batch`, where
`fraction` is the share of layers a worker backpropagates (worker j of k runs
fraction j/k, profile.cpp:89-92). This module measures those rows for a
ChainMlp on a B200 (spb_profile_task: graph-replayed forward + truncated
backward of one worker's batch) and writes them in that schema, so the
reference's simulator can schedule real B200 SPB tasks. The simulator itself
stays on the CPU (out of scope).

Knots are at fraction s/L for s = 1..L (exact layer counts). backward_ms is
made nondecreasing with a running max, the reference's validity rule
(profile.cpp:24-25): a longer suffix never runs faster; only timing noise
could say otherwise.
"""
from typing import List, Sequence

from . import spb

HEADER = "model,fraction,forward_ms,backward_ms,peak_mem_gb,grad_size_mb,batch"


def grad_size_mb(widths: Sequence[int]) -> float:
    """Gradient size in MiB (fp32), as the reference's table lists it."""
    return 4.0 * sum(spb.block_dims(widths)) / float(1 << 20)


def measure(model: str, widths: Sequence[int], batch: int, device: int = 0, reps: int = 10, seed: int = 7) -> List[str]:
    """CSV rows (no header) of one model's profile on the given GPU."""
    widths = list(widths)
    L = len(widths) - 1
    X, Y, W = spb.gen_chain_mlp(widths, max(batch, 256), seed)
    m = spb.ChainMlp(widths, X, Y, W, k=1, per_worker_batch=batch, device=device)
    rows, best_b = [], 0.0
    try:
        for s in range(1, L + 1):
            f, b, mem = m.profile_task(batch, s, reps)
            best_b = max(best_b, b)
            rows.append(f"{model},{s / L:.6g},{f:.4f},{best_b:.4f},{mem:.4f},{grad_size_mb(widths):.3f},{batch}")
    finally:
        m.close()
    return rows


def to_csv(rows: Sequence[str]) -> str:
    return "\n".join([HEADER, *rows]) + "\n"
