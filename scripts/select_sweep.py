#!/usr/bin/env python
"""NEXT-3: the paper's select benchmarks (Figs 4-9) re-run on B200.

Every shape is a Q x n matrix of uniformly random fp32 keys, resident in
HBM.  For each shape we time (CUDA events, after a warm-up):
  * ours   — knn_select (the single-pass select; a cluster per row when Q < #SMs),
  * paper  — knn_select_paper (the paper's quick multi-select as written: repeated
             ballot/popc partitions through global aux arrays, warp per query),
and report ms, ms per query, algorithmic GB/s = (Q n 4 + Q k 8) / t and its fraction of
the HBM peak.  A seeded sample of rows of every shape is checked against the CPU oracle
(bit-exact).  The CPU column of Fig 9 (STL nth_element on one core) is
replaced by the oracle's per-row full sort on one host thread, timed on a few rows.

  python scripts/select_sweep.py [--quick] [--out gpurun_out/select_sweep.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: parity of the sampled rows, CPU timing)
from paper_1309_5478_b200 import knn  # noqa: E402


def shapes(quick):
    out = []
    ks = [64, 128, 256, 512]
    for ln in ([13, 15, 18] if quick else range(13, 19)):          # Fig 4: Q = 8192
        for k in ks:
            out.append(("fig4", 8192, 1 << ln, k))
    for Q in ([1024, 8192, 65536] if quick else [1024, 2048, 4096, 8192, 16384, 32768, 65536]):
        for k in ks:                                                # Fig 5: n = 65536
            out.append(("fig5", Q, 65536, k))
    for lr in ([-3, 5, 13, 17] if quick else [-3, 1, 5, 9, 11, 13, 15, 17]):  # Fig 6: n Q = 2^27
        n = 1 << ((27 + lr) // 2)
        Q = (1 << 27) // n
        for k in ([2, 32, 512] if not quick else [32, 512]):
            if k <= n:
                out.append(("fig6", Q, n, k))
    for Q in ([8, 64, 256] if quick else [8, 16, 32, 64, 128, 256]):  # Fig 8: n = 2^20
        for k in [2, 32, 256, 1024]:
            out.append(("fig8", Q, 1 << 20, k))
    for ln in ([16, 20] if quick else [16, 17, 18, 19, 20]):         # Fig 9: Q = 256
        for k in [2, 16, 128, 1024]:
            out.append(("fig9", 256, 1 << ln, k))
    return out


def timed(fn, reps, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "select_sweep.json"))
    ap.add_argument("--no-paper", action="store_true")
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        peak_src = "measured"
    except Exception:
        peak, peak_src = 6650.0, "fallback"
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    rows = []
    for fig, Q, n, k in shapes(args.quick):
        gen.manual_seed(1309100 + Q * 7 + n)
        D = torch.rand((Q, n), generator=gen, device=dev, dtype=torch.float32)
        nbytes = Q * n * 4 + Q * k * 8
        reps = max(1, min(20, int(2e9 // max(Q * n * 4, 1))))
        ours = timed(lambda: knn.select(D, k), reps)
        kind, splits = knn.last_select_kernel()
        # parity on sampled rows (bit-exact vs the oracle's sort of the same fp32 row)
        g = np.random.Generator(np.random.Philox(Q + n + k))
        sample = np.unique(g.integers(0, Q, size=min(Q, 4)))
        gi, gd = knn.select(D, k)
        Ds = D[torch.from_numpy(sample).to(dev)].cpu().numpy()
        ri, rd = oracle.select_f32(Ds, k)
        ok = bool(np.array_equal(gi[torch.from_numpy(sample).to(dev)].cpu().numpy(), ri) and
                  np.array_equal(gd[torch.from_numpy(sample).to(dev)].cpu().numpy().view(np.uint32),
                                 rd.view(np.uint32)))
        rec = {"fig": fig, "Q": Q, "n": n, "k": k, "ours_ms": ours, "ours_ms_per_query": ours / Q,
               "ours_gbs": nbytes / ours / 1e6, "ours_frac": nbytes / ours / 1e6 / peak,
               "kernel": kind, "splits": splits, "parity_rows": len(sample), "parity_ok": ok}
        if not args.no_paper:
            paper = timed(lambda: knn.select_paper(D, k), max(1, reps // 4))
            pi, pd = knn.select_paper(D, k)
            pok = bool(torch.equal(pi, gi) and torch.equal(pd.view(torch.int32), gd.view(torch.int32)))
            rec.update({"paper_ms": paper, "paper_gbs": nbytes / paper / 1e6,
                        "speedup_vs_paper_kernel": paper / ours, "paper_equal": pok})
        if fig == "fig9":
            R = 2
            Dh = D[:R].cpu().numpy()
            t0 = time.perf_counter()
            oracle.select_f32(Dh, k, threads=1)
            cpu_q = (time.perf_counter() - t0) / R
            rec.update({"cpu_oracle_ms_per_query_1thread": cpu_q * 1e3,
                        "speedup_vs_cpu_1thread": cpu_q * 1e3 / (ours / Q)})
        rows.append(rec)
        print(json.dumps(rec), flush=True)
        del D
        torch.cuda.empty_cache()
    meta = {"peak_gbs": peak, "peak_source": peak_src, "device": torch.cuda.get_device_name(0),
            "data": "U[0,1) fp32 keys (PAPER.md:88), torch Philox seed 1309100 + 7Q + n"}
    json.dump({"meta": meta, "rows": rows}, open(args.out, "w"), indent=1)
    # markdown summary
    md = [f"# Select sweeps (PAPER.md Figs 4-9 shapes) on {meta['device']}", "",
          f"HBM peak {peak:.0f} GB/s ({peak_src}).  ours = knn_select; paper = knn_select_paper "
          "(the paper's quick multi-select, exact ablation).  All sampled rows bit-exact vs the "
          "oracle: " + str(all(r["parity_ok"] for r in rows)) + ".", "",
          "| fig | Q | n | k | kernel | ours ms | ours GB/s | frac | paper ms | ours/paper speedup |",
          "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        md.append(f"| {r['fig']} | {r['Q']} | {r['n']} | {r['k']} | {r['kernel']}"
                  f"{' x' + str(r['splits']) if r['splits'] > 1 else ''} | {r['ours_ms']:.3f} | "
                  f"{r['ours_gbs']:.0f} | {r['ours_frac']:.2f} | "
                  f"{r.get('paper_ms', float('nan')):.3f} | {r.get('speedup_vs_paper_kernel', float('nan')):.1f} |")
    f9 = [r for r in rows if "speedup_vs_cpu_1thread" in r]
    if f9:
        md += ["", "Fig 9 analog (CPU = the oracle's full sort per row, 1 host thread; the paper "
               "used STL nth_element on one core):", "", "| n | k | GPU ms/query | CPU ms/query | speedup |",
               "|---|---|---|---|---|"]
        for r in f9:
            md.append(f"| {r['n']} | {r['k']} | {r['ours_ms_per_query']:.5f} | "
                      f"{r['cpu_oracle_ms_per_query_1thread']:.2f} | {r['speedup_vs_cpu_1thread']:.0f} |")
    open(args.out.replace(".json", ".md"), "w").write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
