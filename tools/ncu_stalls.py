"""Top warp-stall reasons and issue/pipe utilisation of one ncu report.
usage: ncu_stalls.py REP [N]"""
import csv
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
h, v = r[0], r[2]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
get = lambda k: v[h.index(k)] if k in h else "?"
for k in ["gpu__time_duration.sum", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
          "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
          "smsp__average_warp_latency_per_inst_issued.ratio", "smsp__inst_executed.sum", "launch__registers_per_thread",
          "dram__bytes_read.sum", "dram__bytes_write.sum"]:
    print("%-60s %s" % (k, get(k)))
st = [(k, float(v[i] or 0)) for i, k in enumerate(h)
      if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
for k, x in sorted(st, key=lambda t: -t[1])[:n]:
    print("  %-40s %.3f" % (k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), x))
