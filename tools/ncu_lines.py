"""Per-source-line warp-stall samples and executed instructions of an ncu report (read here).

usage: python tools/ncu_lines.py gpurun_out/prof_x.ncu-rep [top]
Also prints the SASS opcode mix (share of executed instructions and of stall samples).
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, agg, op, ops, hdr, why = None, {}, Counter(), Counter(), None, {}
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        try:
            ln = int(r[0])
            w, e = float(r[4] or 0), float(r[7] or 0)
        except (ValueError, IndexError):
            continue
        key = (cur, ln, r[1].strip()[:80])
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += w
        a[1] += e
        if hdr:
            c = why.setdefault(key, Counter())
            for i, h in enumerate(hdr):
                if h.startswith("stall_") and i < len(r):
                    try:
                        c[h[6:]] += float(r[i] or 0)
                    except ValueError:
                        pass
        sass = r[3].split()
        if sass:
            o = sass[1] if sass[0].startswith("@") and len(sass) > 1 else sass[0]
            o = o.split(".")[0]
            op[o] += e
            ops[o] += w
    tw = sum(v[0] for v in agg.values()) or 1
    te = sum(v[1] for v in agg.values()) or 1
    print(f"samples {tw:.0f}  warp instructions {te:.4g}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        rs = ", ".join(f"{n} {c:.0f}" for n, c in why.get(k, Counter()).most_common(3) if c > 0)
        print(f"{v[0] / tw * 100:5.1f}% stall {v[1] / te * 100:5.1f}% inst  {k[0]}:{k[1]}  {k[2][:60]}  [{rs}]")
    to, tso = sum(op.values()) or 1, sum(ops.values()) or 1
    print("opcode mix:")
    for o, c in op.most_common(20):
        print(f"  {o:8s} {c / to * 100:6.2f}% inst {ops[o] / tso * 100:6.2f}% stall")


if __name__ == "__main__":
    main()
