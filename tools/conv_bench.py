"""cfg4 (BASELINE configs[3]): CIFAR10-shaped ConvNet with ResNet18 widths,
k = 8 SPB workers x 128 images, SPB vs full backprop on one B200, plus the
per-class breakdown of one eager step.

    python tools/conv_bench.py [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2111_10672_b200 import spb  # noqa: E402

SHAPE = (32, 32, 3)
CONVS = [(64, 1), (64, 1), (128, 2), (128, 1), (256, 2), (256, 1), (512, 2), (512, 1)]
NOUT, K, BW, N = 10, 8, 128, 8192

if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    X, Y, W = spb.gen_convnet(SHAPE, CONVS, NOUT, N, 7)
    m = spb.ConvNet(SHAPE, CONVS, NOUT, X, Y, W, k=K, per_worker_batch=BW)
    m.set_optimizer(0.01, 0.9, 1e-4)
    out = {"workload": "cfg4: ConvNet 32x32x3, 3x3 convs 64,64,128/2,128,256/2,256,512/2,512 + GAP + head 10, "
                       "k=8 x 128 images", "params": int(sum(spb.convnet_block_dims(SHAPE, CONVS, NOUT)))}
    for full in (False, True):
        m.train_steps(11, 1, 3, full_backprop=full)
        m.synchronize()
        ms = m.time_train_steps(11, 4, steps, full_backprop=full) / steps
        prof, eager = m.profile_step(11, 100, full_backprop=full)
        key = "full" if full else "spb"
        out[key] = {"ms_per_step": round(ms, 4), "samples_per_s": round(K * BW / (ms * 1e-3), 1),
                    "eager_step_ms": round(eager, 3),
                    "phase_ms": {c: round(v["ms"], 3) for c, v in prof.items() if v["launches"]},
                    "gemm_tflops_alg": round(sum(prof[c]["work"] for c in ("gemm_fwd", "gemm_wgrad", "gemm_dgrad"))
                                             / max(1e-9, sum(prof[c]["ms"] for c in ("gemm_fwd", "gemm_wgrad", "gemm_dgrad")))
                                             / 1e9, 1),
                    "launches_per_step": m.launches_per_step()}
    out["spb_speedup"] = round(out["full"]["ms_per_step"] / out["spb"]["ms_per_step"], 4)
    m.close()
    print(json.dumps(out))
