"""Registers / spills per kernel from the ptxas logs of the last build:
python tools/regs.py <source-stem> [name-filter]"""
import re
import subprocess
import sys

log = open(f"build/csrc/{sys.argv[1]}.ptxas.log").read().split("ptxas info    : Compiling entry function")
for blk in log[1:]:
    dem = subprocess.run(["c++filt", blk.split("'")[1]], capture_output=True, text=True).stdout.strip()
    if len(sys.argv) < 3 or sys.argv[2] in dem:
        regs = re.search(r"Used (\d+) registers", blk).group(1)
        spill = re.search(r"(\d+) bytes spill stores", blk).group(1)
        print(f"{regs:>4} regs {spill:>4} B spill  {dem[:110]}")
