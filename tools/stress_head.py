"""Stress aid: repeat the deep-wide step vs partial_backprop comparison and
report the worst per-block relative error per repetition."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10672_b200 import spb  # noqa: E402

widths = [4096] * 8 + [1]
k, bw, N = 8, 16, 1024
X, Y, W = spb.gen_chain_mlp(widths, N, 7)
L = len(widths) - 1
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
bad = 0
for rep in range(reps):
    m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw)
    m.set_optimizer(0.0)
    m.set_fused_update(False)
    m.train_steps(11 + rep, 1, 1)
    agg = m.get_grads()
    batches = m.last_batch(k * bw)
    pgs = [spb.partial_backprop(m, None, batches[(j - 1) * bw:j * bw], spb.suffix_layers(j, k, L))
           for j in range(1, k + 1)]
    ref = spb.aggregate(pgs, k)
    errs = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(agg, ref)]
    worst = max(errs)
    if worst > 1e-5:
        bad += 1
        # fp64 numpy head gradient on the same rows: which side is wrong?
        P = [p.astype(np.float64) for p in m.get_params()]
        h = X[batches].astype(np.float64)
        for l in range(L - 1):
            Wl = P[l][:widths[l + 1] * widths[l]].reshape(widths[l + 1], widths[l])
            h = np.tanh(h @ Wl.T + P[l][widths[l + 1] * widths[l]:])
        WL = P[L - 1][:widths[L] * widths[L - 1]].reshape(widths[L], widths[L - 1])
        d = h @ WL.T + P[L - 1][widths[L] * widths[L - 1]:] - Y[batches].astype(np.float64).reshape(-1, widths[L])
        g = np.concatenate([(d.T @ h / len(batches)).ravel(), d.sum(0) / len(batches)])
        e_agg = float(np.linalg.norm(agg[L - 1] - g) / np.linalg.norm(g))
        e_ref = float(np.linalg.norm(ref[L - 1] - g) / np.linalg.norm(g))
        print("rep", rep, "BAD", ["%.2e" % e for e in errs], "head vs fp64: step %.2e partial %.2e" % (e_agg, e_ref),
              flush=True)
    m.close()
print("reps", reps, "bad", bad)
