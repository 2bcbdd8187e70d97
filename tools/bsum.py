"""Print a one-line summary of a bench.py JSON line read from stdin: tools/bsum.py <label>."""
import json
import sys
label = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r = d.get("roofline") or {}
    print(label, d["config"]["kind"], "value=%.4g" % d["value"], "kernel_ms=", r.get("kernel_ms"), "achieved=",
          r.get("achieved"), r.get("unit"), "frac=", r.get("frac"))
