"""Summarise ptxas -v output (registers / spills per kernel): python tools/ptxas_summary.py [log] [regex]"""
import re
import subprocess
import sys

log = sys.argv[1] if len(sys.argv) > 1 else "paper_2505_13813_b200/_lib/obj/ptxas.log"
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
name = None
spill = ""
for line in open(log):
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = "spill %s/%s" % m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        dem = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"\(.*", "", dem)
        if pat is None or pat.search(dem):
            print("%3s regs  %-16s %s" % (m.group(1), spill, dem))
        name = None
