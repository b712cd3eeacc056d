"""Print the key numbers of bench JSON lines: python tools/showbench.py file.jsonl ..."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        r = d.get("roofline") or {}
        e2e = (d.get("e2e") or {}).get("value")
        print(f"{f}: {d.get('config', {}).get('workload')} value={d.get('value', 0):.4g} ms={d.get('ms_per_step', 0):.4f} "
              f"e2e={e2e if e2e is None else f'{e2e:.4g}'} rel={d.get('rel_l2_vs_reference')} "
              f"roof={r.get('kernel')} {r.get('frac', 0):.3f} clocks={d.get('clocks', {}).get('sm_mhz')}")
        st = d.get("stages_ms")
        if st:
            print("   stages:", {k: round(v, 4) for k, v in st.items()})
        if r.get("fp64_tflops"):
            print("   fp64 TF/s:", round(r["fp64_tflops"], 2))
