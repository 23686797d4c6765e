"""Print selected raw metrics of an ncu report (dev tool):
    python scripts/ncu_grep.py REP.ncu-rep [regex ...]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pats = [re.compile(p) for p in (sys.argv[2:] or [
    r"^l1tex__throughput", r"^l1tex__data_pipe_lsu_wavefronts(_mem_lg)?\.sum$",
    r"^l1tex__t_(sectors|requests)_pipe_lsu_mem_global_op_ld\.sum$",
    r"^l1tex__lsu_writeback_active", r"^l1tex__data_bank", r"^smsp__issue_active\.avg\.pct",
    r"^sm__inst_executed\.sum$", r"^smsp__average_warps_issue_stalled_.*_per_issue_active",
    r"^gpu__time_duration\.sum$", r"^sm__warps_active\.avg\.pct",
    r"^l1tex__m_.*", r"^smsp__inst_executed_op_global_ld\.sum$"])]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr, units, data = r[0], r[1], r[2:]
for row in data:
    name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print("##", name[:60])
    vals = []
    for h, u, v in zip(hdr, units, row):
        if any(p.search(h) for p in pats):
            try:
                fv = float(v.replace(",", ""))
            except ValueError:
                continue
            if "stalled" in h and fv < 0.05:
                continue
            vals.append((h, v, u))
    for h, v, u in vals:
        print(f"  {h} = {v} {u}")
