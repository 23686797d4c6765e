"""Per-kernel roofline table from an ncu metric capture (profiles/).

    python scripts/roofline_table.py OUT.md PEAK_GBS rep.ncu-rep [...]

DRAM GB/s = (dram read + write bytes) / kernel time, fraction of the HBM
peak; first launch of each kernel name per report (cold-cache, serialised
under ncu: shares and ratios, not bench numbers)."""
import csv
import io
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TSCALE = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
          "second": 1.0, "s": 1.0}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main():
    md, peak, reps = sys.argv[1], float(sys.argv[2]), sys.argv[3:]
    lines = ["| kernel | time (us) | DRAM (MB) | DRAM GB/s | of HBM peak | L2 hit % | L2 thru % | "
             "SM thru % | issue active % | warps active % | FP64 pipe % | regs | grid |",
             "|---|" + "---|" * 12]
    seen = {}
    for rep in reps:
        h, u, data = rows(rep)
        col = {k: i for i, k in enumerate(h)}

        def num(r, k):
            v = r[col[k]].replace(",", "")
            return float(v) if v else 0.0
        for r in data:
            name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").split("::")[-1]
            name = name.split("<radix")[0]
            seen[name] = seen.get(name, 0) + 1
            if seen[name] > 1:
                continue
            t = num(r, "gpu__time_duration.sum") * TSCALE.get(u[col["gpu__time_duration.sum"]], 1e-9)
            b = (num(r, "dram__bytes_read.sum") * SCALE.get(u[col["dram__bytes_read.sum"]], 1) +
                 num(r, "dram__bytes_write.sum") * SCALE.get(u[col["dram__bytes_write.sum"]], 1))
            gbs = b / t / 1e9 if t else 0.0
            lines.append(
                f"| {name} | {t * 1e6:.1f} | {b / 1e6:.1f} | {gbs:.0f} | {gbs / peak:.1%} | "
                f"{num(r, 'lts__t_sector_hit_rate.pct'):.0f} | "
                f"{num(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
                f"{num(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
                f"{num(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f} | "
                f"{num(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
                f"{num(r, 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.0f} | "
                f"{int(num(r, 'launch__registers_per_thread'))} | {int(num(r, 'launch__grid_size'))} |")
    with open(md, "w") as fh:
        fh.write(f"<!-- scripts/roofline_table.py, peak {peak:.0f} GB/s (fallback), from "
                 f"{', '.join(reps)} -->\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
