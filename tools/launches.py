"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch).

usage: python tools/launches.py FILE [--agg] [--md OUT.md --title TITLE]
Without --agg: one line per launch (name, ns).  With --agg: per kernel name,
launch count, total and mean time and share of the listed GPU time.
"""
import argparse
import collections
import csv
import re


def short(name):
    name = re.sub(r"\(.*$", "", name)  # drop the parameter list
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return name.replace("void ", "")[:90]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("file")
    ap.add_argument("--agg", action="store_true")
    ap.add_argument("--md")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.file)))
    hdr = [r for r in rows if r and r[0] == "ID"][0]
    i, v = hdr.index("Kernel Name"), hdr.index("Metric Value")
    launches = [(r[i], float(r[v].replace(",", ""))) for r in rows if len(r) > v and r[0] != "ID"]
    if not a.agg:
        for n, t in launches:
            print(short(n), int(t))
        return
    agg = collections.OrderedDict()
    for n, t in launches:
        k = short(n)
        c, s = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, s + t)
    total = sum(s for _, s in agg.values())
    lines = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {s / 1e3:.1f} | {s / c / 1e3:.2f} | {100 * s / total:.1f}% |")
    out = "\n".join(lines)
    print(out)
    if a.md:
        with open(a.md, "w") as f:
            f.write(f"# {a.title}\n\n{out}\n")


if __name__ == "__main__":
    main()
