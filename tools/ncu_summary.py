import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
iid = hdr.index("ID"); kn = hdr.index("Kernel Name"); sec = hdr.index("Section Name"); mn = hdr.index("Metric Name"); mv = hdr.index("Metric Value"); mu = hdr.index("Metric Unit")
keep = {"Duration", "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput",
        "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Issue Slots Busy", "Grid Size", "Block Size", "Waves Per SM", "Dynamic Shared Memory Per Block", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Mem Busy", "Max Bandwidth"}
cur = None
for r in rows[1:]:
    if r[iid] != cur:
        cur = r[iid]
        print("== [%s] %s" % (cur, r[kn][:80]))
    if r[mn] in keep:
        print("   %-40s %s %s" % (r[mn], r[mv], r[mu]))
