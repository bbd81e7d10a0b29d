"""Print the per-size table of bench JSON lines (e.g. gpurun_out/quick_*.json)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    print(f, "value %.3e" % d.get("value", 0), "e2e %.3e" % (d.get("e2e") or {}).get("value", 0))
    ps = d.get("config", {}).get("per_size", {})
    for s, r in ps.items():
        print("  %5s ok %8d alloc %8.2f free %7.2f  %.3f G/s" % (s, r["ok"], r["alloc_us"], r["free_us"],
                                                               r["pairs_per_s"] / 1e9))
