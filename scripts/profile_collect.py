"""Collect the gpu_profile.sh reports into profiles/: the ncu summary, the launch list
summary and traffic.json (dram bytes per launch, the bench's roofline `traffic`).

usage: python scripts/profile_collect.py r01"""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

R = sys.argv[1] if len(sys.argv) > 1 else "r02"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
# report -> the key bench.py looks up
KEYS = {"partition": "dist_tc_kernel", "sample": "dist_tc_kernel_sample", "pivot": "pivot_from_mins_kernel",
        "recompute": "candidate_recompute_kernel", "partition3": "dist_tc_kernel_exact",
        "candsel": "candidate_select_kernel", "prep": "prep_kernel",
        # C4 (k = 1024, quantile pivot): keys distinct from the headline's
        "c4_candsel": "candidate_select_warp_kernel", "c4_pivot": "pivot_from_sample_kernel",
        "c4_sample": "dist_tc_kernel_sample_c4", "c4_partition": "dist_tc_kernel_c4"}
summ, traffic = [], {}
for rep, key in KEYS.items():
    path = os.path.join(G, f"{R}_{rep}.ncu-rep")
    if not os.path.exists(path):
        continue
    summ.append(ncu_summary.summarise(path))
    t = ncu_summary.traffic(path)
    if t:
        traffic[key] = list(t.values())[0]
traffic["_source"] = (f"ncu --set full --clock-control none, one launch each, headline bench command, "
                      f"default plan (single-product pivot partition; dist_tc_kernel_exact = the 3-product "
                      f"partition under KNN_PIVOT1=0) (profiles/{R}_ncu_full_summary.txt)")
with open(os.path.join(P, f"{R}_ncu_full_summary.txt"), "w") as f:
    f.write("\n".join(summ) + "\n")
with open(os.path.join(P, "traffic.json"), "w") as f:
    json.dump(traffic, f, indent=1)
# launch list: per kernel count / total / mean (cold-cache, serialised: shares, not absolutes)
lp = os.path.join(G, f"{R}_launches.csv")
if os.path.exists(lp):
    rows = [r for r in csv.reader(open(lp)) if len(r) > 10]
    h = rows[0]
    iN, iV = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        n = r[iN].split("(")[0]
        agg.setdefault(n, [0, 0.0])
        agg[n][0] += 1
        agg[n][1] += float(r[iV].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(P, f"{R}_launches_summary.txt"), "w") as f:
        f.write(f"ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --steps 2 --warmup 1 "
                f"(3 steps: warm-up + 2 timed)\n")
        f.write("%-90s %5s %12s %10s %6s\n" % ("kernel", "n", "total_us", "mean_us", "share"))
        for n, (c, t) in agg.items():
            f.write("%-90s %5d %12.1f %10.1f %5.1f%%\n" % (n[:90], c, t / 1e3, t / c / 1e3, 100 * t / tot))
    import shutil
    shutil.copy(lp, os.path.join(P, f"{R}_launches.csv"))
print("\n".join(summ))
