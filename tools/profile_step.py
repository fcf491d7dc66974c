"""Runs a few cfg3 SPB steps (graph replays) for ncu captures.

    python tools/profile_step.py [--steps S] [--full]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_10672_b200 import spb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--full", action="store_true")
ap.add_argument("--widths", default="4096x16+1")
args = ap.parse_args()
n, rest = args.widths.split("x")
depth, head = rest.split("+")
widths = [int(n)] * int(depth) + [int(head)]
X, Y, W = spb.gen_chain_mlp(widths, 8192, 7)
m = spb.ChainMlp(widths, X, Y, W, k=8, per_worker_batch=128)
m.set_optimizer(0.01, 0.9, 1e-4)
m.train_steps(11, 1, args.steps, full_backprop=args.full)
m.synchronize()
print("launches/step", m.launches_per_step())
