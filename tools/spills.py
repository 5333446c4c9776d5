"""List the kernels of paper_2307_16652_b200/lib/ptxas.log that spill (bytes stored / loaded)."""
import re
import subprocess
import sys
from pathlib import Path

log = (Path(__file__).resolve().parents[1] / "paper_2307_16652_b200/lib/ptxas.log").read_text().split("\n")
cur = None
for line in log:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and (int(m.group(1)) or int(m.group(2)) or "-a" in sys.argv):
        dn = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        print(m.group(1), m.group(2), dn.split("(")[0][:140])
