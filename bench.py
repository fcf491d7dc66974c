#!/usr/bin/env python
"""SPB training-step throughput on B200 (arXiv 2111.10672), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N --steps K --warmup W

Workload (config.workload): BASELINE.json configs[2]/[4] shape "cfg3" -- the
deep ChainMlp 16 x 4096 (+ scalar head, L = 16), k = 8 SPB workers of
per-worker batch 128 (1024 samples per step), synthetic data from the
reference generator make_random_chain_mlp (model.cpp:208-231, seed 7,
N = 8192), batch draws Rng(11).split(step).split(worker). One "step" = one
SPB-SGD iteration over the whole global batch: forward, truncated backward,
per-layer contributor aggregation, momentum-SGD + weight-decay update. With
N GPUs the 8 workers are dealt out in balanced pairs (j, 9-j); value is the
whole-job samples/s, timed with CUDA events on the step stream, max over
ranks. Weights (2 GB as split pairs) and activations exceed the 126 MB L2,
so no flush is needed between steps.

Also reported: full backprop on the same kernels, the dominant kernel's
roofline (tcgen05 3xTF32 GEMMs, tensor bound) and the update kernel's (HBM),
an end-to-end number through the public C ABI with host batches (pinned)
copied in and the loss copied out every step, and the reference CPU path
(oracle/_ref, the unmodified reference SPB core) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SPB train samples/sec at 1/2/4/8 B200 vs full backprop; % of GEMM/HBM roofline"
UNIT = "samples/s"
CFG3 = dict(workload="cfg3: ChainMlp 16x4096 fp32 (+scalar head, L=16), k=8 SPB workers, batch 128/worker",
            widths=[4096] * 16 + [1], k=8, bw=128, N=8192, data_seed=7, step_seed=11, lr=0.01, momentum=0.9,
            weight_decay=1e-4)
CFG2 = dict(workload="cfg2: MLP 784-512-512-10 fp32, 4 SPB workers time-sliced on 1 GPU, batch 128/worker",
            widths=[784, 512, 512, 10], k=4, bw=128, N=4096, data_seed=7, step_seed=11, lr=0.01, momentum=0.9,
            weight_decay=1e-4)
REF_BW = 2  # reference CPU arm: per-worker samples per step (bounded sample)


NVLINK_GBS = 766.7  # measured: one-peer copy-engine pull / push per direction, 1 GiB (profiles/r01_nvlink_copy_engine.txt)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6553.0), d.get("bf16_tflops", 1661.7), d.get("bf16_tflops_sustained", 1404.0), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        # 200 ms as in the profiling recipe; SPB_CLOCK_MS=0 turns sampling off (perturbation checks only).
        self.ms = int(os.environ.get("SPB_CLOCK_MS", "200"))

    def start(self):
        if self.ms <= 0:
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", str(self.ms), "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": ["sampling off (SPB_CLOCK_MS=0)" if self.ms <= 0 else "nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [x for x in sm if x > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local, dist


def max_over_ranks(dist, x: float) -> float:
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def host_info() -> dict:
    """The host the CPU numbers were taken on."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def bench_config(cfg, world: int) -> dict:
    """The workload description shared by BOTH arms (b200 and reference), so
    the driver's same-config check compares like with like."""
    k = cfg["k"]
    return {"workload": cfg["workload"], "widths": "4096x16+1", "k": k, "per_worker_batch": cfg["bw"],
            "global_batch": k * cfg["bw"], "dataset": cfg["N"], "parallelism": f"spb-dp{world} (workers/rank {k // world})",
            "l2": "inputs exceed L2 (2 GB weights)"}


def cpu_reference(cfg, steps: int, warmup: int, bw: int, threads: int):
    """The unmodified reference SPB core (oracle/_ref: spb.cpp + model.cpp
    compiled from the reference's sources) on cfg's shape with per-worker
    batch `bw`, on data from the reference's OWN generator
    make_random_chain_mlp (model.cpp:208-231, via ref_chain_random) -- so
    this process never loads the B200 library. `threads` workers run
    concurrently (1 = the reference as shipped; > 1 is the k-thread harness,
    legal because its model methods are const and thread-safe,
    model.hpp:21-25). Falls back to the C restatement when _ref is absent.
    Returns (samples/s, kind, threads, sample, ms per step)."""
    from oracle.oracle import REF_SO

    widths, k = cfg["widths"], cfg["k"]
    if os.path.exists(REF_SO):
        from oracle.oracle import Ref, RefModel

        m = RefModel(Ref(), widths, samples=cfg["N"], seed=cfg["data_seed"])
        kind = "reference"
        for s in range(1, warmup + 1):
            m.step(k, k * bw, cfg["lr"], cfg["step_seed"], s, False, threads)
        t = m.time_steps(k, k * bw, cfg["lr"], cfg["step_seed"], warmup + 1, steps, False, threads)
    else:
        from oracle.oracle import Oracle

        o = Oracle()
        kind, threads = "port", 1
        X, Y, W = o.gen_chain_mlp(widths, cfg["N"], cfg["data_seed"])
        for s in range(1, warmup + 1):
            o.spb_step(widths, X, Y, W, k, k * bw, cfg["lr"], cfg["step_seed"], s)
        t0 = time.perf_counter()
        for s in range(warmup + 1, warmup + 1 + steps):
            o.spb_step(widths, X, Y, W, k, k * bw, cfg["lr"], cfg["step_seed"], s)
        t = time.perf_counter() - t0
    value = steps * k * bw / t
    sample = (f"{steps} SPB step(s) of {cfg['workload'].split(':')[0]} (widths 4096x16+1, k={k}) with {bw} sample(s) "
              f"per worker ({k * bw} samples/step) after {warmup} warm-up, fp64, plain SGD x -= lr g (the reference's "
              f"only update rule), {threads} worker thread(s); the reference's cost is per sample (per-sample loop "
              f"spb.cpp:63) plus a per-step allocation of each worker's gradient, included here")
    return value, kind, threads, sample, 1e3 * t / steps


def run_reference_arm(args, world, rank):
    cfg = CFG3
    if rank != 0:
        return
    threads = max(1, min(cfg["k"], os.cpu_count() or 1))
    value, kind, cores, sample, ms = cpu_reference(cfg, max(1, args.steps), max(0, args.warmup), REF_BW, threads)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (the reference's own generator make_random_chain_mlp, seed 7)",
            "config": bench_config(cfg, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                             "host": host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def median_profile(m, seed, step0, full, reps=3):
    """Per-class median of `reps` eager profiled steps (spb_profile_step)."""
    runs = [m.profile_step(seed, step0 + i, full_backprop=full) for i in range(reps)]
    med = {}
    for c in runs[0][0]:
        ms = sorted(r[0][c]["ms"] for r in runs)[reps // 2]
        med[c] = dict(runs[0][0][c], ms=ms)
    return med, sorted(r[1] for r in runs)[reps // 2]


def roofline_of(prof: dict, peaks, traffic=None):
    """Roofline of the dominant kernel, the forward GEMM (largest share of the
    step; the kernel profiles/r01_gemm_fwd_ncu_full.json captures for
    `traffic`): algorithmic FLOPs per launch / average launch time from the
    eager profiled step (CUDA events on its stream). 3xTF32 issues 3 tf32
    MMAs per algorithmic MAC and tf32 runs at half the bf16 rate, so the
    tensor-pipe work is 6x the algorithmic FLOPs, compared with the measured
    dense bf16 peak. All GEMM classes together and the HBM-bound update are
    reported beside it."""
    hbm, bf16, bf16_sus, src = peaks

    def rate(classes):
        ms = sum(prof[c]["ms"] for c in classes)
        fl = sum(prof[c]["work"] for c in classes)
        n = sum(prof[c]["launches"] for c in classes)
        return (fl / (ms * 1e-3) / 1e12 if ms > 0 else 0.0), fl, ms, n

    fwd_tf, fwd_fl, fwd_ms, fwd_n = rate(("gemm_fwd",))
    all_tf, all_fl, all_ms, all_n = rate(("gemm_fwd", "gemm_wgrad", "gemm_dgrad"))
    upd = prof["update"]
    upd_gbs = upd["work"] / (upd["ms"] * 1e-3) / 1e9 if upd["ms"] > 0 else 0.0
    return {
        "bound": "tensor", "kernel": f"forward GEMM: {FWD_KERNEL} (tcgen05.mma cta_group::2 kind::tf32, 3xTF32)",
        "achieved": round(6.0 * fwd_tf, 2), "peak": bf16, "unit": "TFLOP/s", "frac": round(6.0 * fwd_tf / bf16, 4),
        "traffic": traffic,
        "peak_source": f"{src} bf16_tflops (burst): every launch of the profiled step is timed alone (serialised, "
                       f"CUDA events on its stream); sustained bf16 = {bf16_sus}",
        "achieved_note": "tensor-pipe TFLOP/s = 6 x algorithmic fp32 GEMM TFLOP/s (3 tf32 products per MAC, tf32 = bf16/2)",
        "algorithmic_tflops": round(fwd_tf, 2), "algorithmic_gflop_per_launch": round(fwd_fl / max(fwd_n, 1) / 1e9, 3),
        "avg_launch_ms": round(fwd_ms / max(fwd_n, 1), 4), "launches_per_step": fwd_n,
        "all_gemms": {"algorithmic_tflops": round(all_tf, 2), "pipe_tflops": round(6.0 * all_tf, 2),
                      "frac": round(6.0 * all_tf / bf16, 4), "launches_per_step": all_n,
                      "note": "forward + wgrad + dgrad; wgrad includes the optimizer epilogue of the fused (<= 512-row) layers"},
        "update_kernel": {"bound": "hbm", "achieved": round(upd_gbs, 1), "peak": hbm, "unit": "GB/s",
                          "frac": round(upd_gbs / hbm, 4) if hbm else None, "bytes_per_step": upd["work"],
                          "ms_per_step": round(upd["ms"], 4), "launches_per_step": upd["launches"],
                          "traffic_bytes_per_step": upd["work"] * 28.0 / 20.0,
                          "note": "the per-layer update kernels of the unfused layers; achieved counts the algorithmic "
                                  "20 B/param (read w, g, mom; write w, mom -- BASELINE.md section 4); the weights' "
                                  "exact 3xTF32 split-pair storage moves 28 B/param (traffic_bytes_per_step)"},
    }


FWD_KERNEL = "gemm_tf32x3_2sm_kernel<0,0,0,240,0>"  # the cfg3 forward GEMM the planner ships


def traffic_from_profiles():
    """dram__bytes_read + write per launch of the SHIPPED forward kernel, from
    the committed `ncu --set full` capture of that same kernel
    (profiles/r02_gemm_fwd_ncu_full.json, tools/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", "r02_gemm_fwd_ncu_full.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            if FWD_KERNEL in d.get("kernel", "").replace(" ", ""):
                return d.get("dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            return None
    return None


def spb_savings(widths, k, bw, world):
    """Backward FLOPs and gradient-exchange bytes of one SPB step vs full
    backprop (north_star: SPB saves both). Backward per layer l over its
    contributor rows: wgrad 2*rows*n_l*n_{l-1}, dgrad 2*rows*n_l*n_{l-1} for
    l >= 2 over the contributor rows of layer l-1 (the rows Delta_{l-1} is
    needed for). Exchange: per layer, the gradient bytes of
    every rank hosting a contributor (a rank without contributors sends
    nothing); at 1 GPU, the bytes of the local aggregate."""
    from paper_2111_10672_b200 import spb

    L = len(widths) - 1
    chunks = spb.layer_chunks(k, L)
    out = {}
    for full in (False, True):
        fl = 0.0
        by = 0.0
        plan = spb.bucket_plan(k, L, max(world, 1), full) if world > 1 else None
        for l in range(1, L + 1):
            m = k if full else chunks[l - 1]
            rows = m * bw
            fl += 2.0 * rows * widths[l] * widths[l - 1]
            if l >= 2:
                fl += 2.0 * (k if full else chunks[l - 2]) * bw * widths[l] * widths[l - 1]
            nranks_l = len(plan[l - 1][2]) if plan else 1
            by += 4.0 * (widths[l] * widths[l - 1] + widths[l]) * nranks_l
        out["full" if full else "spb"] = (fl, by)
    return {"backward_flops_spb": out["spb"][0], "backward_flops_full": out["full"][0],
            "exchange_bytes_spb": out["spb"][1], "exchange_bytes_full": out["full"][1],
            "saved_backward_flops_frac": round(1 - out["spb"][0] / out["full"][0], 4),
            "saved_exchange_bytes_frac": round(1 - out["spb"][1] / out["full"][1], 4)}


CFG4 = dict(workload="cfg4: ConvNet 32x32x3 (CIFAR10 shape), 3x3 convs at ResNet18 widths "
                     "64,64,128/2,128,256/2,256,512/2,512 + global avg pool + head 10, k=8 SPB workers, batch 128/worker",
            shape=(32, 32, 3), convs=[(64, 1), (64, 1), (128, 2), (128, 1), (256, 2), (256, 1), (512, 2), (512, 1)],
            nout=10, k=8, bw=128, N=8192, data_seed=7, step_seed=11, lr=0.01, momentum=0.9, weight_decay=1e-4)


def _measure_sub(m, c, out, world, dist, K, W_):
    """SPB vs full backprop on one model: CUDA events on the step stream, max over ranks."""
    for full in (False, True):
        m.set_params(m.initial_params())
        m.train_steps(c["step_seed"], 1, W_, full_backprop=full)
        m.synchronize()
        barrier(dist)
        ms = m.time_train_steps(c["step_seed"], 1 + W_, K, full_backprop=full)
        barrier(dist)
        ms = max_over_ranks(dist, ms)
        prof, _ = m.profile_step(c["step_seed"], 1000, full_backprop=full)
        gemm_ms = sum(prof[q]["ms"] for q in ("gemm_fwd", "gemm_wgrad", "gemm_dgrad"))
        gemm_fl = sum(prof[q]["work"] for q in ("gemm_fwd", "gemm_wgrad", "gemm_dgrad"))
        out["full_backprop" if full else "spb"] = {
            "value": round(K * c["k"] * c["bw"] / (ms * 1e-3), 2), "unit": UNIT, "ms_per_step": round(ms / K, 4),
            "launches_per_step": m.launches_per_step(),
            "gemm_alg_tflops": round(gemm_fl / max(gemm_ms, 1e-9) / 1e9, 1),
            "phase_ms": {q: round(prof[q]["ms"], 3) for q in prof if prof[q]["launches"]}}
    out["spb_speedup"] = round(out["spb"]["value"] / out["full_backprop"]["value"], 4)
    return out


def run_cfg4(world, rank, local, dist, K, W_):
    """BASELINE configs[3] on the same engine: SPB vs full backprop samples/s
    and the eager per-class breakdown. Reported beside the cfg3 headline."""
    from paper_2111_10672_b200 import spb

    c = CFG4
    X, Y, W = spb.gen_convnet(c["shape"], c["convs"], c["nout"], c["N"], c["data_seed"])
    m = spb.ConvNet(c["shape"], c["convs"], c["nout"], X, Y, W, k=c["k"], per_worker_batch=c["bw"], device=local)
    if world > 1:
        m.comm_init_torch(dist, rank, world)
    m.set_optimizer(c["lr"], c["momentum"], c["weight_decay"])
    out = {"workload": c["workload"], "params": int(sum(spb.convnet_block_dims(c["shape"], c["convs"], c["nout"]))),
           "data": "synthetic (numpy uniform images/targets, seed 7)",
           "lowering": "implicit GEMM via TMA im2col (c_in % 32 == 0) on tcgen05 3xTF32; the RGB layer's forward as a direct fp32 kernel (its wgrad over im2col columns of the contributor samples); dgrad / wgrad on two streams; wgrads of >= 256 output channels on the CTA pair"}
    _measure_sub(m, c, out, world, dist, K, W_)
    barrier(dist)
    m.close()
    return out


def run_cfg2(world, rank, local, dist, K, W_):
    """BASELINE configs[1] (the reference's MLP, 4 workers time-sliced on ONE
    B200) on the same engine. With N ranks it runs as N independent replicas
    (the configuration is a 1-GPU one: no exchange; value = all replicas'
    samples/s, max-over-ranks time); the 4 workers spread over the ranks with
    the exchange are reported beside it (`sharded`, N <= k): a 0.67 M-param
    model whose step is ~0.1 ms, so there the per-layer exchange latency
    dominates."""
    from paper_2111_10672_b200 import spb

    c = CFG2
    X, Y, W = spb.gen_chain_mlp(c["widths"], c["N"], c["data_seed"])
    out = {"workload": c["workload"], "data": "synthetic (reference generator make_random_chain_mlp, seed 7)",
           "reference_cpu_samples_per_s_1core": "834 SPB / 636 full (BASELINE.md section 2, survey container)"}
    m = spb.ChainMlp(c["widths"], X, Y, W, k=c["k"], per_worker_batch=c["bw"], device=local)
    m.set_optimizer(c["lr"], c["momentum"], c["weight_decay"])
    _measure_sub(m, c, out, world, dist, K, W_)
    barrier(dist)
    m.close()
    if world > 1:
        out["multi_gpu"] = f"replicas only: {world} independent 1-GPU steps (configs[1] is a 1-GPU configuration)"
        for key in ("spb", "full_backprop"):
            out[key]["value"] = round(out[key]["value"] * world, 2)
        if world <= c["k"]:
            m = spb.ChainMlp(c["widths"], X, Y, W, k=c["k"], per_worker_batch=c["bw"], device=local)
            m.comm_init_torch(dist, rank, world)
            m.set_optimizer(c["lr"], c["momentum"], c["weight_decay"])
            sh = {"note": f"the 4 workers spread over {world} ranks with the per-layer exchange ({m.comm_mode})"}
            _measure_sub(m, c, sh, world, dist, K, W_)
            barrier(dist)
            m.close()
            out["sharded"] = sh
    return out


def run_b200(args, world, rank, local, dist):
    from paper_2111_10672_b200 import spb

    cfg = CFG3
    widths, k, bw = cfg["widths"], cfg["k"], cfg["bw"]
    L = len(widths) - 1
    X, Y, W = spb.gen_chain_mlp(widths, cfg["N"], cfg["data_seed"])
    m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw, device=local)
    del W
    comm_mode = None
    if world > 1:
        m.comm_init_torch(dist, rank, world)
        comm_mode = m.comm_mode
    workers = spb.rank_workers(k, L, rank, world) if world > 1 else list(range(1, k + 1))
    rows = len(workers) * bw
    m.set_optimizer(cfg["lr"], cfg["momentum"], cfg["weight_decay"])
    if os.environ.get("SPB_FUSED") is not None:  # optimizer placement 0 / 1 / 2 (default 2)
        m.set_fused_update(int(os.environ["SPB_FUSED"]))
    seed = cfg["step_seed"]
    W_ = max(3, args.warmup)
    K = max(1, args.steps)

    clocks = ClockSampler(local)
    clocks.start()
    # SPB: warm-up, then K timed steps (graph replays, CUDA events on the step stream).
    m.train_steps(seed, 1, W_)
    m.synchronize()
    barrier(dist)
    ms = m.time_train_steps(seed, 1 + W_, K)
    barrier(dist)
    ms = max_over_ranks(dist, ms)
    launches = m.launches_per_step()
    # Full backprop on the same kernels (baseline_estimate, spb.cpp:149-160).
    m.set_params(m.initial_params())
    m.train_steps(seed, 1, W_, full_backprop=True)
    m.synchronize()
    barrier(dist)
    ms_full = m.time_train_steps(seed, 1 + W_, K, full_backprop=True)
    barrier(dist)
    ms_full = max_over_ranks(dist, ms_full)
    clk = clocks.stop()

    # Per-kernel-class timings of one eager step (roofline numerator).
    # Median over 3 profiled steps per class: one eager step is at the mercy
    # of the power-capped clock of the moment.
    prof, prof_step_ms = median_profile(m, seed, 1000, False)
    prof_full, _ = median_profile(m, seed, 1010, True)

    # End to end through the public C ABI: pinned host batches in, loss out.
    e2e = None
    try:
        import torch

        nb = 4
        Xp = torch.empty((nb, rows, widths[0]), dtype=torch.float32).pin_memory()
        Yp = torch.empty((nb, rows, widths[-1]), dtype=torch.float32).pin_memory()
        for i in range(nb):
            idx = np.concatenate([spb.draw_batch(seed, 5000 + i, j, bw, cfg["N"]) for j in workers])
            Xp[i].copy_(torch.from_numpy(X[idx]))
            Yp[i].copy_(torch.from_numpy(Y[idx]))
        xs = [Xp[i].numpy() for i in range(nb)]
        ys = [Yp[i].numpy() for i in range(nb)]
        losses = np.zeros(max(K, W_), dtype=np.float32)
        for i in range(W_):
            m.step_host(xs[i % nb], ys[i % nb])
        barrier(dist)
        t0 = time.perf_counter()
        for i in range(K):
            loss = m.step_host(xs[i % nb], ys[i % nb])
        m.synchronize()
        t_sync = time.perf_counter() - t0
        barrier(dist)
        t_sync = max_over_ranks(dist, t_sync)
        # The headline e2e: the same public-API step, pipelined (the next
        # batch's H2D copy overlaps this step; losses copied back per step).
        for i in range(W_):
            m.step_host_async(xs[i % nb], ys[i % nb], losses[i:i + 1])
        m.synchronize()
        barrier(dist)
        t0 = time.perf_counter()
        for i in range(K):
            m.step_host_async(xs[i % nb], ys[i % nb], losses[i:i + 1])
        m.synchronize()
        t_e2e = time.perf_counter() - t0
        barrier(dist)
        t_e2e = max_over_ranks(dist, t_e2e)
        e2e = {"value": K * k * bw / t_e2e, "unit": UNIT, "h2d_bytes_per_step": rows * (widths[0] + widths[-1]) * 4 * world,
               "d2h_bytes_per_step": 4 * world, "ms_per_step": 1e3 * t_e2e / K,
               "path": "spb_step_host_async (C ABI): pinned host rows H2D on a copy stream (double-buffered) + graph "
                       "step + per-step loss D2H, synchronised at the end",
               "synchronous": {"value": K * k * bw / t_sync, "ms_per_step": 1e3 * t_sync / K,
                               "path": "spb_step_host: H2D + step + loss D2H + host sync every step"},
               "last_loss": float(losses[K - 1]), "last_loss_sync": loss}
    except Exception as ex:  # noqa: BLE001
        e2e = {"value": None, "unit": UNIT, "error": repr(ex)}

    value = K * k * bw / (ms * 1e-3)
    full_value = K * k * bw / (ms_full * 1e-3)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W_,
        "ms_per_step": round(ms / K, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (3xTF32 tcgen05)", "data": "synthetic (reference generator make_random_chain_mlp, seed 7)",
        "config": bench_config(cfg, world),
        "engine": {"optimizer": "momentum 0.9, wd 1e-4, lr 0.01", "aggregation": comm_mode or "local (1 GPU)",
                   "graph_chain": (max(1, min(16, int(os.environ["SPB_CHAIN"]))) if "SPB_CHAIN" in os.environ
                                   else 1)},
        "spb_savings": spb_savings(widths, k, bw, world),
        "full_backprop": {"value": round(full_value, 2), "unit": UNIT, "ms_per_step": round(ms_full / K, 4),
                          "spb_speedup": round(value / full_value, 4)},
        "gpu_launches": launches * K,
        "launches_per_step": launches,
        "clocks": clk,
        "e2e": e2e,
        "roofline": roofline_of(prof, load_peaks(), traffic_from_profiles()),
        # (world > 1: "nvlink" added below -- this rank's exchange bytes per step
        # over the step time, against the measured one-peer copy bandwidth)
        "phase_ms": {c: round(prof[c]["ms"], 3) for c in prof},
        "phase_ms_full_backprop": {c: round(prof_full[c]["ms"], 3) for c in prof_full},
        "eager_step_ms": round(prof_step_ms, 3),
    }
    if world > 1:
        comm_bytes = max_over_ranks(dist, float(prof["comm"]["work"]))
        step_s = ms / K * 1e-3
        nv = comm_bytes / step_s / 1e9
        line["roofline"]["nvlink"] = {
            "bound": "nvlink", "achieved": round(nv, 1), "peak": NVLINK_GBS, "unit": "GB/s",
            "frac": round(nv / NVLINK_GBS, 4), "bytes_per_step": comm_bytes,
            "note": f"{comm_mode}: bytes this rank pulls (p2p / rh), pushes + pulls (push: gradient rows stored to "
                    "their owners, weight rows pulled) or reduces (nccl buckets, algorithmic) per step, "
                    "max over ranks, averaged over the whole step; peak = measured one-peer copy-engine bandwidth "
                    "per direction (profiles/r01_nvlink_copy_engine.txt)"}
    barrier(dist)
    m.close()
    del m
    if not args.no_conv:
        try:
            line["cfg4_convnet"] = run_cfg4(world, rank, local, dist, min(K, 10), W_)
        except Exception as ex:  # noqa: BLE001
            line["cfg4_convnet"] = {"error": repr(ex)}
    try:
        line["cfg2_mlp"] = run_cfg2(world, rank, local, dist, K, W_)
    except Exception as ex:  # noqa: BLE001
        line["cfg2_mlp"] = {"error": repr(ex)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference is single-threaded -> 1 core is
        # the baseline; the k-thread harness (one worker per thread) beside it.
        v, kind, cores, sample, _ = cpu_reference(cfg, 1, 0, 1, 1)
        v8, _, t8, sample8, _ = cpu_reference(cfg, 1, 0, REF_BW, max(1, min(cfg["k"], os.cpu_count() or 1)))
        line["cpu_baseline"] = {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                                "host": host_info(),
                                "threaded_harness": {"value": round(v8, 3), "cores": t8, "sample": sample8}}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-conv", action="store_true", help="skip the cfg4 ConvNet sub-measurement")
    args = ap.parse_args()
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference_arm(args, world, rank)
        return
    world, rank, local, dist = dist_setup(args)
    try:
        run_b200(args, world, rank, local, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
