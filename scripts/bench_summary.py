"""Print the essentials of a bench.py JSON line (file argument)."""
import json
import sys

b = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
r = b["roofline"]
e = b.get("e2e") or {}
print("value %.4e pts/s  ms/step %.3f  n_gpus %s  e2e %s  plan %s" % (
    b["value"], b["ms_per_step"], b["n_gpus"], e.get("value") and "%.3e" % e["value"], r["plan"]))
print("dominant %s avg %.3f ms frac %.3f (sust %.3f) achieved %.1f %s step_floor_frac %s" % (
    r["kernel"], r["avg_launch_ms"], r["frac"], r.get("frac_sustained", 0), r["achieved"], r["unit"],
    r.get("step_floor_frac")))
for o in r["others"]:
    print("  other %s avg %.3f ms frac %.3f achieved %.1f %s" % (o["kernel"][:60], o["avg_launch_ms"], o["frac"],
                                                              o["achieved"], o["unit"]))
print("share", {k: round(v, 3) for k, v in r["step_share"].items()}, "clocks", b["clocks"])
