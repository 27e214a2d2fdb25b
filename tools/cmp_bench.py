"""Print step time, roofline fraction and per-kernel times of bench JSON lines
(one file per argument; the last line of each is used)."""
import json, sys
for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable:", e); continue
    r = d["roofline"]
    km = {k: round(v * 1e3, 1) for k, v in r.get("kernel_ms", {}).items()}
    print(f"{p}: {d['value']:.4e} {d['ms_per_step']:.4f} ms frac {r['frac']:.4f} "
          f"step_frac {r.get('step_frac', 0):.4f} us {km} sm {d['clocks']['sm_mhz']}")
