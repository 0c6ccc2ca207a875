"""Summarise an ncu report (raw page) into the metrics DESIGN.md / bench.py cite.

usage: python scripts/ncu_summary.py report.ncu-rep [more.ncu-rep ...] > summary.txt"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    r"^Kernel Name$", r"^gpu__time_duration.sum$", r"^dram__bytes_read.sum$", r"^dram__bytes_write.sum$",
    r"^gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed$",
    r"^sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed$",
    r"^sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active$",
    r"^lts__throughput.avg.pct_of_peak_sustained_elapsed$", r"^lts__t_sector_hit_rate.pct$",
    r"^sm__throughput.avg.pct_of_peak_sustained_elapsed$", r"^smsp__issue_active.avg.pct_of_peak_sustained_active$",
    r"^sm__warps_active.avg.pct_of_peak_sustained_active$", r"^launch__registers_per_thread$",
    r"^launch__grid_size$", r"^launch__block_size$", r"^launch__cluster_dim_x$",
    r"^launch__shared_mem_per_block_dynamic$", r"^sm__cycles_elapsed.avg.per_second$",
    r"^smsp__inst_executed.sum$",
]


def summarise(path):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"== {path}"]
    for vals in rows[2:]:
        for pat in KEYS:
            for h, u, v in zip(hdr, units, vals):
                if re.search(pat, h):
                    out.append(f"  {h} = {v} {u}".rstrip())
        out.append("  --")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarise(p))


def traffic(path):
    """{kernel base name: dram read+write bytes per launch} from one report."""
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    out = {}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        name = re.sub(r"^void ", "", d["Kernel Name"]).split("(")[0].split("::")[-1].split("<")[0]
        tot = sum(float(d[m]) * scale[u[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        out[name] = tot
    return out
