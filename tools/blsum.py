"""Print the key fields of bench.py JSON lines: python tools/blsum.py FILE..."""
import json
import sys

for fn in sys.argv[1:]:
    for line in open(fn):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        print(f"== {fn}: {d['config']['plan']} {d['ms_per_step']*1e3:.1f} us/step  speedup={d.get('speedup_vs_default')}"
              f"  clocks={d.get('clocks', {}).get('sm_mhz')}")
        print("   ", {k: round(v["ms_per_step"] * 1e3, 1) for k, v in d["kernels"].items()})
        pt = d["config"].get("plan_times_us")
        if pt and any(v for v in pt.values()):
            print("    plan times", {k: round(v, 1) for k, v in pt.items() if v})
