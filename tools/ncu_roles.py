"""Stall reasons per warp role of a warp-specialised kernel (read here from an ncu --set full report).

usage: python tools/ncu_roles.py rep.ncu-rep
Roles are split at the setmaxnreg instructions (USETMAXREG.TRY_ALLOC / DEALLOC) in SASS order."""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 4 and r[0].startswith("0x")]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
cuts = [i for i, r in enumerate(data) if "USETMAXREG" in r[1]] + [len(data)]
start = 0
for k, end in enumerate(cuts):
    seg = data[start:end]
    agg = collections.Counter()
    ins = 0
    for r in seg:
        ins += int(r[5] or 0)
        for c in cols:
            agg[hdr[c]] += int(r[c] or 0)
    tot = sum(agg.values()) or 1
    print(f"segment {k} (SASS rows {start}-{end}): {ins:.3e} warp instructions, {tot} samples: " +
          ", ".join(f"{h[6:]} {100 * v / tot:.0f}%" for h, v in agg.most_common(6)))
    start = end
