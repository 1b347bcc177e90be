"""Per-kernel mean duration and DRAM bytes from an ncu --csv launch list
captured with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
(tools/README.md).  Usage: python tools/launch_table.py launches.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, mi, vi, ui, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[start + 1:]:
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1.0)
        per[(r[idi], r[ki].split("(")[0])][r[mi]] = v * scale
    agg = collections.defaultdict(list)
    for (_, k), m in per.items():
        agg[k].append(m)
    tot = sum(m.get("gpu__time_duration.sum", 0.0) for ms in agg.values() for m in ms)
    for k, ms in sorted(agg.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1])):
        t = sum(m.get("gpu__time_duration.sum", 0.0) for m in ms)
        rd = sum(m.get("dram__bytes_read.sum", 0.0) for m in ms) / len(ms)
        wr = sum(m.get("dram__bytes_write.sum", 0.0) for m in ms) / len(ms)
        print(f"{k[-48:]:48s} n={len(ms):4d} mean={t / len(ms):10.2f} us  share={t / tot:.3f}  "
              f"dram r/w per launch {rd / 1e9:.3f} / {wr / 1e9:.3f} GB  -> {(rd + wr) / (t / len(ms)) / 1e3:.0f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1])
