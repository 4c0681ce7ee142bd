"""Print the key fields of bench.py JSON lines (value, e2e, roofline, clocks)."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    r = d.get("roofline", {})
    print(f"== {f}: value {d.get('value'):.4g} ms/step {d.get('ms_per_step', 0):.3f} e2e {d.get('e2e', {}).get('value', 0):.4g} launches {d.get('gpu_launches')} clocks {d.get('clocks')}")
    print("   ", {k: (round(r[k], 4) if isinstance(r.get(k), float) else r.get(k)) for k in
                  ['frac', 'pair_kernel_ms_per_step', 'sample_kernel_ms_per_step', 'leaf_ms', 'levels_ms', 'compose_gather_ms']})
    if d.get("cpu_baseline"):
        print("    cpu", d["cpu_baseline"]["value"])
