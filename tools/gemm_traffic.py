"""Build profiles/r01_gemm_traffic.json (feeds bench.py's roofline.traffic) from one eager C2 wave.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/launches.csv \
        python tools/profile_step.py --M 4 --steps 1 --eager --gemm-log gpurun_out/gemm_log.json
    python tools/gemm_traffic.py gpurun_out/launches.csv gpurun_out/gemm_log.json > profiles/r01_gemm_traffic.json

The eager step issues one libspx GEMM launch per logged call, so the n-th gemm_bf16_kernel launch
in the ncu list is the n-th entry of the GEMM log.
"""
import collections
import csv
import json
import sys


def key_of(entry):
    if entry[0] == "group":
        return str(("group", tuple(tuple(x) for x in entry[1]), entry[2], entry[3]))
    return str(tuple(entry))


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    log = json.load(open(sys.argv[2]))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    idi, ki, mi, vi, ui = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    launches: dict = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or "gemm_bf16_kernel" not in r[ki]:
            continue
        d = launches.setdefault(int(r[idi]), {})
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        elif r[ui] in ("Kbyte", "KB"):
            v *= 1e3
        elif r[ui] in ("Mbyte", "MB"):
            v *= 1e6
        elif r[ui] in ("Gbyte", "GB"):
            v *= 1e9
        d[r[mi]] = v
    seq = list(launches.values())
    if len(seq) != len(log):
        raise SystemExit(f"{len(seq)} GEMM launches in the ncu list but {len(log)} logged GEMM calls")
    agg = collections.OrderedDict()
    for entry, d in zip(log, seq):
        a = agg.setdefault(key_of(entry), [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a[2] += d.get("gpu__time_duration.sum", 0.0)
    out = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     "--clock-control none, tools/profile_step.py --M 4 --steps 1 --eager --gemm-log "
                     "(cold cache, serialised)",
           "per_shape": {k: {"launches": n, "dram_bytes_per_launch": round(b / n), "ncu_us": round(t / n, 2)}
                         for k, (n, b, t) in agg.items()}}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
