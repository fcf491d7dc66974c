"""Prints the key fields of a bench.py JSON line (stdin)."""
import json
import sys

for line in sys.stdin:
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r = d.get("roofline", {})
    print(f"value={d.get('value')} ms/step={d.get('ms_per_step')} full={d.get('full_backprop', {}).get('value')} "
          f"full_ms={d.get('full_backprop', {}).get('ms_per_step')} gemm_frac={r.get('frac')} "
          f"alg_tflops={r.get('algorithmic_tflops')} e2e={(d.get('e2e') or {}).get('value')}")
    print("  phase", d.get("phase_ms"))
    print("  phase_full", d.get("phase_ms_full_backprop"))
