"""Timeline of the cfg3 SPB step as replayed from one chained CUDA graph
(spb_trace_steps: %globaltimer stamps around every op, per stream), per rank.

    python tools/trace.py [world] [modes, e.g. p2p,nccl] [chain] [widths] [full]
    python tools/trace.py summary gpurun_out/trace_*.npz

Writes gpurun_out/trace_<mode>_w<world>_c<chain>[_full]_r<rank>.npz and prints
a per-stream / per-class summary.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CLS = {0: "fwd", 1: "wgrad", 2: "dgrad", 3: "head", 4: "colred", 5: "update", 6: "gather", 7: "comm", 100: "wait"}


def stream_name(s):
    if s >= 20:
        return f"wpull{s - 20}"
    if s >= 10:
        return f"gpull{s - 10}"
    return {0: "main", 1: "wgrad", 2: "upd", 3: "split", 4: "coll"}.get(s, f"s{s}")


def summary(path):
    d = np.load(path)
    t0, t1, cls, st, sub = d["t0"], d["t1"], d["cls"], d["stream"], d["sub"]
    nsub = int(sub.max()) + 1
    # step boundaries: the first forward GEMM of each step (the gather may run
    # early: it does not wait for the previous step's weights)
    g = sorted(min(t0[(cls == 0) & (sub == k)]) for k in range(nsub) if ((cls == 0) & (sub == k)).any())
    span = (t1.max() - t0.min()) / 1e6
    print(f"== {os.path.basename(path)}: {len(t0)} ops, {nsub} steps, {span:.3f} ms "
          f"({span / nsub:.3f} ms/step); forward starts (ms): {[round(float(x) / 1e6, 3) for x in g]}")
    if len(g) >= 2:
        print(f"   steady step period (forward start to forward start): {np.diff(g).mean() / 1e6:.3f} ms")
    rows = {}
    for c, s, a, b in zip(cls, st, t0, t1):
        k = (stream_name(s), CLS.get(int(c), str(c)))
        r = rows.setdefault(k, [0, 0.0])
        r[0] += 1
        r[1] += (b - a) / 1e6
    for (s, c), (n, ms) in sorted(rows.items()):
        print(f"   {s:8s} {c:8s} n={n:4d} total {ms:8.3f} ms  ({ms / nsub:.3f}/step)")
    # a middle step's op sequence
    m = nsub // 2
    sel = np.where(sub == m)[0]
    sel = sel[np.argsort(t0[sel])]
    base = t0[sel].min()
    print(f"   step {m} ops (start ms rel. to its first op, dur us):")
    line = []
    for i in sel:
        line.append(f"{stream_name(st[i])}:{CLS.get(int(cls[i]), cls[i])}@{(t0[i] - base) / 1e6:.3f}+{(t1[i] - t0[i]) / 1e3:.0f}")
    for j in range(0, len(line), 6):
        print("     " + "  ".join(line[j:j + 6]))


def run(rank, world, port, mode, chain, widths_s, full):
    import torch.distributed as dist

    from paper_2111_10672_b200 import spb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if world > 1:
        os.environ["SPB_COMM"] = mode
        dist.init_process_group("gloo", rank=rank, world_size=world)
    n, rest = widths_s.split("x")
    depth, head = rest.split("+")
    widths = [int(n)] * int(depth) + [int(head)]
    X, Y, W = spb.gen_chain_mlp(widths, 8192, 7)
    m = spb.ChainMlp(widths, X, Y, W, k=8, per_worker_batch=128, device=rank)
    if world > 1:
        m.comm_init_torch(dist, rank, world)
    m.set_optimizer(0.01, 0.9, 1e-4)
    m.train_steps(11, 1, 5, full_backprop=full)
    m.synchronize()
    if world > 1:
        dist.barrier()
    tr = m.trace_steps(11, 6, chain, full_backprop=full)
    tag = f"{mode if world > 1 else 'local'}_w{world}_c{chain}{'_full' if full else ''}_r{rank}"
    out = os.path.join(ROOT, "gpurun_out", f"trace_{tag}.npz")
    np.savez(out, **tr)
    if world > 1:
        dist.barrier()
    m.close()
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        summary(out)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "summary":
        for p in sys.argv[2:]:
            summary(p)
        sys.exit(0)
    import torch.multiprocessing as mp

    world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["p2p"]
    chain = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    widths = sys.argv[4] if len(sys.argv) > 4 else "4096x16+1"
    full = len(sys.argv) > 5 and sys.argv[5] == "full"
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for i, md in enumerate(modes):
        mp.start_processes(run, args=(world, 29800 + 10 * i + world, md, chain, widths, full), nprocs=world,
                           start_method="spawn")
