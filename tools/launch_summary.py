"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name.

    python tools/launch_summary.py gpurun_out/launches.csv [--md out.md] [--title ...]
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--md")
    ap.add_argument("--title", default="launch list")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1e3 if u in ("ns", "nsecond") else (v if u in ("us", "usecond") else v * 1e3)
        nm = r[ki].split("(")[0].replace("void ", "")
        agg[nm][0] += 1
        agg[nm][1] += v
    tot = sum(x[1] for x in agg.values())
    lines = [f"# {a.title}", "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    lines.append(f"| **total** | {sum(c for c, _ in agg.values())} | {tot:.1f} | 100% |")
    out = "\n".join(lines) + "\n"
    print(out)
    if a.md:
        open(a.md, "w").write(out)


if __name__ == "__main__":
    main()
