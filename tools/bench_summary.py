"""Short table of a bench.py JSON line (main record + sub-records)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])


def row(name, r):
    rf = r.get("roofline") or {}
    e = r.get("e2e") or {}
    c = r.get("config") if isinstance(r.get("config"), dict) else {}
    print(f"{name:8s} value {r['value'] / 1e6:9.1f} M/s  mean {r['ms_per_step']:9.3f} ms  median {rf.get('dominant_ms', 0):9.3f} ms  "
          f"frac {rf.get('frac', 0):.3f}  e2e {e.get('ms_per_step', 0):9.3f} ms  launches {r.get('gpu_launches')}  "
          f"plan_s {r.get('plan_s', c.get('plan_s'))}  clocks {r.get('clocks', {}).get('sm_mhz')} {r.get('clocks', {}).get('reasons')}")


row("main", d)
for k, v in (d.get("configs") or {}).items():
    row(k, v)
ra = d.get("e2e_reference_api")
if ra:
    print("reference_api", {k: ra[k] for k in ("ms_per_step", "first_call_ms", "value") if k in ra})
print("cpu_baseline", d.get("cpu_baseline"))
