"""Registers / spills per kernel from `python -m paper_2512_09642_b200.build -v --force` output on stdin.
usage: python -m paper_2512_09642_b200.build -v --force 2>&1 | python tools/ptxas_regs.py [REGEX]"""
import re
import sys

pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
fn = None
spill = ""
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line) or re.search(r"Function properties for (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = "%s/%s" % m.groups()
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and fn and (pat is None or pat.search(fn)):
        t = re.search(r"(k\w+?)I(L[^E]*E(?:L[^E]*E)*)", fn)
        name = (t.group(1) + "<" + ",".join(re.findall(r"L\w(\d+)E", t.group(2))) + ">") if t else fn[-40:]
        print("%-24s regs %4s spill %s" % (name, m.group(1), spill))
