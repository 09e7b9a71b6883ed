"""Registers / spills per kernel from a ptxas -v log.  usage: ptxas_regs.py build/x.ptxas.log [substring]"""
import re, subprocess, sys

log = open(sys.argv[1]).read().split("ptxas info    : Compiling entry function")
sub = sys.argv[2] if len(sys.argv) > 2 else ""
for b in log[1:]:
    name = b.split("'")[1]
    dm = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    if sub in dm:
        m = re.search(r"Used (\d+) registers", b)
        sp = re.search(r"(\d+) bytes spill stores", b)
        print(f"{dm[:100]:100s} regs {m.group(1) if m else '?':>4s} spill {sp.group(1) if sp else '?'}")
