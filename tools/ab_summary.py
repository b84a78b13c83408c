"""Summarise bench A/B lines: solve time, loop launch, roofline fraction, loop phase cycles."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    r = d["roofline"]
    k = d["kernels"]["richardson_loop"]
    ph = {a: b for a, b in k["phase_cycles_per_iter"].items() if not isinstance(b, dict)}
    print(f, f"value {d['value'] * 1e3:.4f} ms  loop {r['launch_us']:.1f} us  frac {r['frac']:.4f}", ph,
          k["phase_cycles_per_iter"].get("apply_split"), k["phase_cycles_per_iter"].get("sync_split"))
