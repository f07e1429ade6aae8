"""Print the interesting parts of a bench JSON line (stdin) compactly."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        print(line[:300])
        continue
    d = json.loads(line)
    r = d.get("roofline") or {}
    print(f"{d['config'].get('workload')}: {d['value']:.1f} {d['unit']} ms/step {d.get('ms_per_step')} "
          f"e2e {d.get('e2e', {}).get('value')} clocks {d.get('clocks')}")
    print(f"  roofline {r.get('kernel')} {r.get('bound')} achieved {r.get('achieved')} peak {r.get('peak')} frac {r.get('frac')}")
    for k, v in (r.get("by_kernel") or {}).items():
        print(f"    {k}: {json.dumps(v)}")
    print(f"  plan {json.dumps(d.get('plan'))}")
    if d.get("cpu_baseline"):
        print(f"  cpu {json.dumps(d['cpu_baseline'])[:400]}")
