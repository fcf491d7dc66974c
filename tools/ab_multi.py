"""A/B of per-context environment knobs at N GPUs (run under torchrun): for
each round and variant, every rank builds the cfg3 context with the variant's
environment set, joins the exchange, and times SPB and full-backprop graph
steps (CUDA events, max over ranks). Knobs read once per process
(SPB_PLACEMENT, SPB_COMM_SMS read at comm_init is fine) must not be varied.

    torchrun --nproc-per-node 4 tools/ab_multi.py [--conv] ROUNDS name=ENV:VAL,ENV:VAL [name=...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from paper_2111_10672_b200 import spb

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    args = sys.argv[1:]
    conv = args[0] == "--conv"  # cfg4 (the ConvNet) instead of cfg3
    if conv:
        args = args[1:]
    rounds = int(args[0])
    variants = []
    for spec in args[1:]:
        name, _, envs = spec.partition("=")
        variants.append((name, dict(e.split(":", 1) for e in envs.split(",") if e)))
    widths, k, bw = [4096] * 16 + [1], 8, 128
    shape, convs = (32, 32, 3), [(64, 1), (64, 1), (128, 2), (128, 1), (256, 2), (256, 1), (512, 2), (512, 1)]
    if conv:
        X, Y, W = spb.gen_convnet(shape, convs, 10, 8192, 7)
    else:
        X, Y, W = spb.gen_chain_mlp(widths, 8192, 7)
    res = {}
    for r in range(rounds):
        for name, env in variants:
            saved = {key: os.environ.get(key) for key in env}
            os.environ.update(env)
            if conv:
                m = spb.ConvNet(shape, convs, 10, X, Y, W, k=k, per_worker_batch=bw, device=local)
            else:
                m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw, device=local)
            m.comm_init_torch(dist, rank, world)
            m.set_optimizer(0.01, 0.9, 1e-4)
            out = {}
            for full in (False, True):
                m.set_params(W)
                m.train_steps(11, 1, 5, full_backprop=full)
                m.synchronize()
                dist.barrier()
                ms = m.time_train_steps(11, 6, 20, full_backprop=full) / 20
                t = torch.tensor([ms])
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                out["full" if full else "spb"] = round(float(t[0]), 4)
            dist.barrier()
            m.close()
            for key, v in saved.items():
                if v is None:
                    os.environ.pop(key, None)
                else:
                    os.environ[key] = v
            res.setdefault(name, []).append(out)
            if rank == 0:
                print(json.dumps({"round": r, "variant": name, "env": env, **out}), flush=True)
    if rank == 0:
        summ = {n: {"spb_ms": [d["spb"] for d in v], "full_ms": [d["full"] for d in v],
                    "spb_samples_per_s_best": round(k * bw / (min(d["spb"] for d in v) * 1e-3), 1)}
                for n, v in res.items()}
        print(json.dumps({"world": world, "summary": summ}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
