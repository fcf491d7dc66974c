"""Same-process A/B of the dgrad TMEM chunk (spb_set_gemm_chunk) on the cfg3
SPB step: alternating settings, fresh context each (graphs are captured with
the setting active), 20 timed graph steps after 5 warm-up, momentum + wd.

    python tools/ab_chunk.py [rounds]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10672_b200 import spb  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
widths, k, bw, N = [4096] * 16 + [1], 8, 128, 8192
X, Y, W = spb.gen_chain_mlp(widths, N, 7)
lib = spb.load_library()
res = {}
for r in range(rounds):
    for ck in (4, 2):
        lib.spb_set_gemm_chunk(1, ck)
        m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw)
        m.set_optimizer(0.01, 0.9, 1e-4)
        for full in (False, True):
            m.set_params(W)
            m.train_steps(11, 1, 5, full_backprop=full)
            m.synchronize()
            ms = m.time_train_steps(11, 6, 20, full_backprop=full) / 20
            res.setdefault(f"dgrad_chunk{ck}_{'full' if full else 'spb'}", []).append(round(ms, 4))
        m.close()
lib.spb_set_gemm_chunk(1, 0)
print(json.dumps(res))
