"""Print the key numbers of bench.py JSON lines in log files."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if line.startswith("pcg plan"):
            print(f, line.strip())
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        k = d.get("kernel_ms_per_step") or {}
        print(f, "value %.1f e2e %s pcg_it %s pcg_ms %s frac %s" % (
            d["value"], (d.get("e2e") or {}).get("value"), d.get("pcg_iterations_per_step"), k.get("pcg"),
            (d.get("roofline") or {}).get("frac")), {a: round(b, 4) for a, b in k.items()})
