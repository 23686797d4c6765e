"""Top SASS lines by warp-stall samples from an ncu report's source page
(dev tool): python scripts/source_hotspots.py REP KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
data = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr) and r[0] != "Address"]
half = len(data) // 2 if len(data) % 2 == 0 and data[:len(data) // 2] == data[len(data) // 2:] else len(data)
data = data[:half]
f = lambda x: float(x) if x not in ("", "-") else 0.0
iw, ie, it, isrc = (hdr.index(k) for k in ("Warp Stall Sampling (All Samples)",
                                            "Instructions Executed", "Avg. Threads Executed",
                                            "Source"))
tot = sum(f(r[iw]) for r in data) or 1.0
inst = sum(f(r[ie]) for r in data)
print(f"instructions executed {inst:.3e}, stall samples {tot:.0f}")
print("| stall % | executed | threads | SASS |\n|---|---|---|---|")
for r in sorted(data, key=lambda r: -f(r[iw]))[:top]:
    print(f"| {f(r[iw]) / tot * 100:.1f} | {r[ie]} | {r[it]} | `{r[isrc].strip()[:70]}` |")
