"""Summarises an `ncu --set full` capture (exported with `ncu -i X.ncu-rep
--page raw --csv`) into the JSON kept under profiles/: the kernel's name,
duration, DRAM bytes per launch (dram__bytes_read + write: bench.py's
roofline.traffic), tensor-pipe and DRAM utilisation, registers, occupancy.

    python tools/ncu_summary.py RAW.csv OUT.json "source command" [algorithmic_bytes] [algorithmic_flops]
"""
import csv
import json
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def to_bytes(v, unit):
    return float(v) * SCALE.get(unit, 1)


def main(raw, out, source, alg_bytes=None, alg_flops=None):
    rows = list(csv.reader(open(raw)))
    head, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        kernels.append({k: (d[k] + (" " + units[head.index(k)] if units[head.index(k)] else "")).strip()
                        for k in KEYS if k in d})
        dr = to_bytes(d["dram__bytes_read.sum"], units[head.index("dram__bytes_read.sum")])
        dw = to_bytes(d["dram__bytes_write.sum"], units[head.index("dram__bytes_write.sum")])
        kernels[-1]["dram_bytes"] = dr + dw
    k0 = kernels[0]
    res = {"source": source, "kernel": k0["Kernel Name"].split("(")[0].replace("void ", ""), "kernels": kernels,
           "dram_bytes_per_launch": k0["dram_bytes"]}
    if alg_bytes:
        res["algorithmic_bytes_per_launch"] = float(alg_bytes)
    if alg_flops:
        res["algorithmic_flops_per_launch"] = float(alg_flops)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: res[k] for k in ("kernel", "dram_bytes_per_launch")}))


if __name__ == "__main__":
    main(*sys.argv[1:])
