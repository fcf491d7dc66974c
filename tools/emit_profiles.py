"""Writes B200 task profiles in the reference simulator's schema
(profile.hpp:64-67) for the cfg1/cfg3/cfg5 MLPs.

    python tools/emit_profiles.py [out.csv]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_10672_b200 import jigsaw_profiles as jp  # noqa: E402

MODELS = [
    ("MLP-784-512-512-10", [784, 512, 512, 10], 128),
    ("ChainMlp-16x1024", [1024] * 16 + [1], 128),
    ("ChainMlp-16x2048", [2048] * 16 + [1], 128),
    ("ChainMlp-16x4096", [4096] * 16 + [1], 128),
    ("ChainMlp-16x8192", [8192] * 16 + [1], 128),
]

if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/b200_profiles.csv"
    rows = []
    for name, widths, batch in MODELS:
        rows += jp.measure(name, widths, batch, reps=10)
        print(rows[-1], flush=True)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as f:
        f.write(jp.to_csv(rows))
    print("wrote", out)
