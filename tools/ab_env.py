"""A/B of environment knobs on one box: each variant runs in a fresh process
(graphs are captured with the knob active), variants alternate over rounds.

    python tools/ab_env.py cfg3|cfg4 rounds name=ENV:VAL,ENV:VAL [name=...]

cfg3: SPB and full-backprop graph-step ms (20 steps after 5 warm-up, momentum +
wd); cfg4: the ConvNet's (10 steps after 3)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(workload):
    sys.path.insert(0, ROOT)
    from paper_2111_10672_b200 import spb

    out = {}
    if workload == "cfg3":
        widths, k, bw, N = [4096] * 16 + [1], 8, 128, 8192
        X, Y, W = spb.gen_chain_mlp(widths, N, 7)
        m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw)
        steps, warm = 20, 5
    else:
        shape, convs = (32, 32, 3), [(64, 1), (64, 1), (128, 2), (128, 1), (256, 2), (256, 1), (512, 2), (512, 1)]
        X, Y, W = spb.gen_convnet(shape, convs, 10, 8192, 7)
        m = spb.ConvNet(shape, convs, 10, X, Y, W, k=8, per_worker_batch=128)
        steps, warm = 10, 3
    m.set_optimizer(0.01, 0.9, 1e-4)
    for full in (False, True):
        m.set_params(W)
        m.train_steps(11, 1, warm, full_backprop=full)
        m.synchronize()
        out["full" if full else "spb"] = m.time_train_steps(11, 1 + warm, steps, full_backprop=full) / steps
    prof, _ = m.profile_step(11, 100)
    out["phase_ms"] = {c: round(v["ms"], 3) for c, v in prof.items() if v["launches"]}
    print(json.dumps(out))


def main():
    workload, rounds = sys.argv[1], int(sys.argv[2])
    variants = []
    for spec in sys.argv[3:]:
        name, _, envs = spec.partition("=")
        env = dict(e.split(":", 1) for e in envs.split(",") if e)
        variants.append((name, env))
    res = {}
    for r in range(rounds):
        for name, env in variants:
            e = dict(os.environ, **env)
            p = subprocess.run([sys.executable, __file__, "--child", workload], env=e, capture_output=True, text=True)
            try:
                d = json.loads(p.stdout.strip().splitlines()[-1])
            except Exception:  # noqa: BLE001
                d = {"error": p.stderr[-500:]}
            res.setdefault(name, []).append(d)
    summary = {n: {"spb_ms": [round(d.get("spb", -1), 4) for d in v], "full_ms": [round(d.get("full", -1), 4) for d in v],
                   "phase_ms": v[-1].get("phase_ms"), "error": v[-1].get("error")} for n, v in res.items()}
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2])
    else:
        main()
