"""Summarise an ncu --set full report (per kernel launch): duration, tensor-pipe and XU activity,
issue activity, DRAM bytes.  Reads `ncu -i <rep> --page raw --csv` output.

    ncu -i rep.ncu-rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv [--md out.md]
"""
import csv
import sys

COLS = [("gpu__time_duration.sum", "us", 1e-3),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %", 1),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU %", 1),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1),
        ("dram__bytes_read.sum", "DRAM rd MB", 1e-6),
        ("dram__bytes_write.sum", "DRAM wr MB", 1e-6),
        ("gpc__cycles_elapsed.avg.per_second", "GHz", 1e-9)]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h, units = rows[0], rows[1]
    idx = {n: i for i, n in enumerate(h)}
    out = ["| kernel | " + " | ".join(c[1] for c in COLS) + " |", "|---" * (len(COLS) + 1) + "|"]
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0][:60]
        vals = []
        for col, _, sc in COLS:
            i = idx.get(col)
            if i is None:
                vals.append("-")
                continue
            try:
                v = float(r[i].replace(",", ""))
                u = units[i]
                if col.startswith("gpu__time"):
                    sc = {"usecond": 1, "msecond": 1e3, "nsecond": 1e-3, "second": 1e6}.get(u, 1)
                if col.startswith("dram__bytes") and u in ("Mbyte", "MB"):
                    sc = 1
                if col.startswith("dram__bytes") and u in ("Gbyte", "GB"):
                    sc = 1e3
                if col.startswith("dram__bytes") and u in ("Kbyte", "KB"):
                    sc = 1e-3
                if col.startswith("gpc__") and u in ("Ghz", "GHz", "cycle/nsecond"):
                    sc = 1
                vals.append(f"{v * sc:.2f}")
            except ValueError:
                vals.append(r[i])
        out.append(f"| `{name}` | " + " | ".join(vals) + " |")
    txt = "\n".join(out)
    if len(sys.argv) > 3 and sys.argv[2] == "--md":
        open(sys.argv[3], "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
