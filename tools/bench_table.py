"""One line per bench JSON: step ms, Gproducts/s, numeric ms/frac, per-pass ms."""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(p, "ERR", e)
        continue
    pm = {k: round(v, 3) for k, v in d.get("pass_ms", {}).items()}
    print(f"{d['config']['workload'][:10]:10s} step={d['ms_per_step']:.3f}ms {d['value'] / 1e9:6.1f} Gp/s "
          f"num={d['numeric_ms']:.3f}ms frac={d['roofline']['frac']:.3f} launches={d['gpu_launches']} {pm}")
