"""Summarise ncu --set full reports (raw page) into a text table and a JSON
record per kernel: duration, dram bytes read/write, DRAM/SM throughput %,
registers, occupancy, L2 hit rate.  usage: ncu_raw_summary.py OUT_JSON REP..."""
import csv
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct"]
out = {}
for rep in sys.argv[2:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        rec = {}
        for w in WANT:
            if w in h:
                v = r[h.index(w)].replace(",", "")
                u = units[h.index(w)]
                try:
                    v = float(v)
                except ValueError:
                    pass
                rec[w] = [v, u]
        out[name] = rec
        print("== %s  (%s)" % (name, rep))
        for k, (v, u) in rec.items():
            print("   %-58s %s %s" % (k, v, u))
json.dump(out, open(sys.argv[1], "w"), indent=1)
