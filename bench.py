#!/usr/bin/env python
"""Headline benchmark (BASELINE.json "metric"): k-NNG points/s at N=65536, d=256, k=32.

A step is one pass of the whole hot path over the workload: row norms + split (a-S2),
distance GEMM (a-S3) and per-row select (a-S4) for all N query rows; under torchrun the
query rows are sharded over the ranks (Par-1: rank 0's points are broadcast, results
all-gathered, both inside the step).  Inputs are resident in HBM when a step starts;
L2 is flushed (256 MiB write, untimed) before every timed step.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config H|C1..C5]

Prints ONE JSON line on rank 0 (see DESIGN.md §Measurement for every field)."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "k-NNG points/sec at N=65536,d=256,k=32 (1/2/4/8 B200); select GB/s; GEMM tensor util"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=150)  # ~0.5 s timed: enough nvidia-smi clock samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="H", help="H (headline) or C1..C5")
    ap.add_argument("--plan", default="auto", choices=["auto", "materialised"])
    ap.add_argument("--shard", default="auto", choices=["auto", "sym", "query", "corpus"],
                    help="multi-GPU sharding (knn_graph_sharded / knn_search_sharded); auto: sym for "
                         "the k-NNG (corpus for C5, BASELINE configs[4]), query rows for search")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU seconds of the oracle cpu_baseline sample")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "bf16_tflops": p["bf16_tflops"],
                "bf16_tflops_sustained": p.get("bf16_tflops_sustained", p["bf16_tflops"]),
                "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback"}


def get_config(name):
    from paper_1309_5478_b200 import datagen
    return datagen.HEADLINE if name == "H" else datagen.CONFIGS[name]


def workload_name(cfg):
    mode = "k-NNG" if cfg.mode == "graph" else f"k-NN search M={cfg.M}"
    return f"{mode} N={cfg.N} d={cfg.d} k={cfg.k} {cfg.dist} fp32 (squared L2)"


# ------------------------------------------------------------------ clocks ----------
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,power.draw,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, smax, reasons, n_load = [], None, set(), 0
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                clk, mx, util = float(parts[0]), float(parts[1]), float(parts[2])
            except ValueError:
                continue
            smax = mx
            if util >= 50:
                n_load += 1
                sm.append(clk)
                for nm, v in zip(names, parts[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples_under_load": n_load}


# ------------------------------------------------------------------ CPU oracle ------
def oracle_rows_per_s(X, k, graph, target_s, threads, Q=None):
    """Time the oracle (as it stands) on a bounded sample of query rows (of Q, default X)."""
    import numpy as np
    import oracle
    Q = X if Q is None else Q
    N = Q.shape[0]
    g = np.random.Generator(np.random.Philox(4242))
    rows = g.choice(N, size=min(N, threads), replace=False)
    t0 = time.perf_counter()
    oracle.knn(Q, X, k, rows=rows, graph=graph, threads=threads, want_r32=False)
    t1 = time.perf_counter() - t0
    R = int(min(N, max(len(rows), len(rows) * target_s / max(t1, 1e-3))))
    R = max(threads, (R // threads) * threads)
    rows = g.choice(N, size=min(N, R), replace=False)
    t0 = time.perf_counter()
    oracle.knn(Q, X, k, rows=rows, graph=graph, threads=threads, want_r32=False)
    dt = time.perf_counter() - t0
    return len(rows) / dt, len(rows), dt


def run_reference(args):
    """--impl reference: the oracle, as it stands, on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import oracle
    from paper_1309_5478_b200 import datagen
    cfg = get_config(args.config)
    Q, X = datagen.config_inputs(cfg)
    threads = oracle.default_threads()
    graph = cfg.mode == "graph"
    # one step = a bounded sample of the workload's query rows (same rows every step)
    g = np.random.Generator(np.random.Philox(4243))
    per_step = max(threads, 2 * threads)
    rows = g.choice(cfg.M, size=min(cfg.M, per_step), replace=False)

    def step():
        oracle.knn(Q, X, cfg.k, rows=rows, graph=graph, threads=threads, want_r32=False)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = len(rows) * args.steps / dt
    sample = (f"{len(rows)} seeded query rows of the {cfg.M}-row workload per step "
              f"(fp64 direct distances to all {cfg.N} points + full std::sort per row)")
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(cfg), "N": cfg.N, "d": cfg.d, "k": cfg.k,
                   "sample_rows_per_step": len(rows)},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ ours ------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1309_5478_b200 import datagen, knn, sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # KNN_BENCH_SHARE_GPU=1 (testing the multi-rank flow on a one-GPU box): every rank on
    # cuda:0, gloo for the host-side collectives; never used for a reported number
    share = os.environ.get("KNN_BENCH_SHARE_GPU", "0") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # host-side plumbing (id exchange, barriers, max over ranks) on gloo; the data path's
        # collectives are the library's: NCCL over NVLink (its init log on, so the ranks'
        # communicator is visible), or the host transport when the ranks share one GPU
        if not share:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("gloo")
        sharded.init(transport="host" if share else "nccl")
    cfg = get_config(args.config)
    search = cfg.mode != "graph"  # C3: k-NN search of M queries against N corpus points
    N, d, k = cfg.N, cfg.d, cfg.k
    M = cfg.M if search else N  # rows (queries) of the job
    X_host = datagen.points(N, d, cfg.dist, cfg.seed) if rank == 0 else None
    X = torch.from_numpy(X_host).to(dev) if rank == 0 else torch.empty((N, d), device=dev)
    Q_host = (datagen.points(M, d, cfg.dist, cfg.seed + 1000) if rank == 0 else None) if search else X_host
    Q = (torch.from_numpy(Q_host).to(dev) if rank == 0 else torch.empty((M, d), device=dev)) if search else X
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2

    # sharding: k-NNG -> the ranks split the upper triangle (Par-3, the transpose reuse
    # survives sharding), C5 -> corpus columns + all-to-all + k-way merge (BASELINE
    # configs[4]); search -> query rows (Par-1).  One GPU runs the same call as one rank.
    shard = args.shard
    if shard == "auto":
        shard = "query" if search else ("corpus" if cfg.sharding == "corpus" else "sym")
    if search and shard == "sym":
        raise SystemExit("--shard sym is a k-NNG mode")
    out_i = torch.empty((M, k), dtype=torch.int32, device=dev)
    out_d = torch.empty((M, k), dtype=torch.float32, device=dev)

    def step():
        if search:
            return sharded.search(Q, X, k, mode=shard, out=(out_i, out_d))
        return sharded.graph(X, k, mode=shard, out=(out_i, out_d))

    def barrier():
        if world > 1:
            dist.barrier()

    assert knn.gemm_path() == 0 or os.environ.get("KNN_GEMM") == "simt", "tensor-core path expected"
    knn.set_plan({"auto": knn.PLAN_AUTO,
                  "materialised": knn.PLAN_MATERIALISED}[args.plan])
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.15)
    knn.profile_enable(True)
    launches0 = knn.launch_count()
    stream = torch.cuda.current_stream()
    total_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()  # evict L2 (untimed)
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        barrier()
        torch.cuda.synchronize()
        total_ms += e0.elapsed_time(e1)
    launches = knn.launch_count() - launches0
    shard_ran = {0: "query", 1: "corpus", 2: "sym"}.get(knn.last_shard_mode(), "none")
    sym_shard = shard_ran == "sym" and world > 1
    prof = {kname: knn.profile_read(kname) for kname in knn.KERNELS}
    knn.profile_enable(False)
    clocks = sampler.stop()

    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = M / (ms_per_step / 1e3)  # points (query rows) per second, whole job

    # ---- roofline of the dominant kernel (per-launch averages over the timed region)
    peaks = load_peaks()
    lo_r, hi_r = sharded.block_range(M, world, rank)
    R_local = hi_r - lo_r
    # this rank's share of the work: query rows x all N points, or (corpus sharding) all M
    # rows x its column block; the symmetric plans multiply the upper triangle only
    if shard_ran == "corpus":
        c_lo, c_hi = sharded.block_range(N, world, rank)
        rows_w, cols_w = M, c_hi - c_lo
    else:
        rows_w, cols_w = R_local, N
    d_pad = -(-d // 64) * 64
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f)
    except Exception:
        traffic = {}

    plan_code = knn.last_plan()
    S_samp = knn.pivot_sample_size(cols_w, k)  # the library's own sample size (N / 8..16)

    # committed ncu captures: the headline's kernels under their names, C4's GEMMs with a
    # "_c4" suffix (profiles/traffic.json)
    def tkey(kernel):
        return kernel + "_c4" if args.config == "C4" and kernel.startswith("dist_tc_kernel") else kernel

    # plans 5 / 6: the k <= 32 partition ran on the single hi.hi product (chosen on the
    # device, or KNN_PIVOT1=1) and the candidate select re-evaluated the survivors in fp32
    # (DESIGN.md §6.5); 3 / 4: the FP32-accurate 3-product partition
    pivot1 = plan_code in (5, 6)
    sym_plan = plan_code in (2, 3, 5)
    pivot_plan = plan_code in (3, 4, 5, 6)

    def pairs_of(kernel):
        if kernel == "dist_tc_kernel_sample":
            return rows_w * S_samp
        if sym_plan:
            # symmetric: the upper triangle of 256x256 blocks (split over the ranks by Par-3)
            nblk = -(-N // 256)
            return nblk * (nblk + 1) / 2 * 256.0 * 256.0 / (world if sym_shard else 1)
        return rows_w * cols_w

    # Peak: the measured BURST bf16 (= fp16) dense rate — the timed region is well under a
    # second, so the sustained (power-capped, 4 s) figure would flatter the kernel; the
    # sustained fraction is reported beside it.
    def tensor_roof(name, kernel, ms, n, products=3):
        avg = ms / max(n, 1)
        pairs = pairs_of(kernel)
        flop = products * 2.0 * pairs * d_pad  # executed fp16 tensor flop (3 products: split)
        useful = 2.0 * pairs * d  # the dot products the method needs (triangle for the k-NNG)
        r = {"kernel": name, "bound": "tensor", "achieved": flop / (avg * 1e-3) / 1e12,
             "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
             "peak_kind": f"fp16 dense = bf16 {peaks['source']} burst",
             "useful_tflops": useful / (avg * 1e-3) / 1e12, "avg_launch_ms": avg,
             "launches": n, "flop_per_launch": flop, "traffic": traffic.get(tkey(kernel)),
             "traffic_source": traffic.get("_source")}
        r["frac"] = r["achieved"] / r["peak"]
        r["frac_sustained"] = r["achieved"] / peaks["bf16_tflops_sustained"]
        return r

    def hbm_roof(name, kernel, ms, n, bytes_per_launch):
        avg = ms / max(n, 1)
        r = {"kernel": name, "bound": "hbm", "achieved": bytes_per_launch / (avg * 1e-3) / 1e9,
             "peak": peaks["hbm_gbs"], "unit": "GB/s", "avg_launch_ms": avg, "launches": n,
             "algorithmic_bytes": bytes_per_launch, "traffic": traffic.get(kernel),
             "traffic_source": traffic.get("_source")}
        r["frac"] = r["achieved"] / r["peak"]
        return r

    rooflines = []
    f_ms, f_n = prof["fused"]
    g_ms, g_n = prof["gemm"]
    s_ms, s_n = prof["select"]
    m_ms, m_n = prof["merge"]
    p_ms, p_n = prof["prep"]
    x_ms, x_n = prof["xmerge"]
    if f_n and pivot_plan:
        rooflines.append((f_ms, tensor_roof(
            "dist_tc_kernel<PIVOT%s%s> (a-S5: GEMM with the quickselect partition in its epilogue%s)"
            % ("1" if pivot1 else "", ",SYM" if plan_code in (3, 5) else "",
               ", single hi.hi product" if pivot1 else ""), "dist_tc_kernel", f_ms, f_n,
            products=1 if pivot1 else 3)))
    if g_n and pivot_plan:
        gr = tensor_roof("dist_tc_kernel<MINS> (pivot sample pass: rows x N/div sampled columns (div 8-16 by N) -> 32-column chunk minima)"
                         if k <= 32 else
                         f"dist_tc_kernel<SAMPLE> (quantile-pivot sample: single-product upper bounds, rows x {S_samp} columns)",
                         "dist_tc_kernel_sample", g_ms, g_n, products=1)
        rooflines.append((g_ms, gr))
    elif g_n:
        gr = tensor_roof("dist_tc_kernel (a-S3)", "dist_tc_kernel", g_ms, g_n)
        if plan_code == 0:  # blocked: the launches split the rows
            gl = max(g_n // args.steps, 1)
            for key in ("achieved", "useful_tflops", "flop_per_launch", "frac", "frac_sustained"):
                gr[key] /= gl
        if plan_code == 2:
            # the symmetric GEMM does half the MMA work and writes the whole matrix: its
            # binding roofline is the HBM write of D (+ operand reads)
            avg = g_ms / g_n
            dbytes = rows_w * (-(-N // 4) * 4) * 4.0 + 2 * N * d_pad * 4.0
            gr["tensor_frac"] = gr["frac"]
            gr.update({"bound": "hbm", "achieved": dbytes / (avg * 1e-3) / 1e9,
                       "peak": peaks["hbm_gbs"], "unit": "GB/s", "algorithmic_bytes": dbytes,
                       "peak_kind": f"HBM {peaks['source']} copy bandwidth"})
            gr["frac"] = gr["achieved"] / gr["peak"]
            gr["kernel"] = "dist_tc_kernel<SYM> (a-S3, symmetric k-NNG: upper triangle, direct + transposed stores)"
        rooflines.append((g_ms, gr))
    piv_rows = R_local if sym_shard else rows_w
    if s_n and pivot_plan:
        if k <= 32:
            rooflines.append((s_ms, hbm_roof("pivot_from_mins_kernel (pivot = k-th smallest of the row's chunk minima)",
                                             "pivot_from_mins_kernel", s_ms, s_n,
                                             piv_rows * (S_samp // 32 * 4.0 + 8.0))))
        else:
            rooflines.append((s_ms, hbm_roof("pivot_from_sample_kernel (pivot = bucketed order statistic of the sample)",
                                             "pivot_from_sample_kernel", s_ms, s_n, piv_rows * (S_samp * 4.0 + 4.0))))
    elif s_n:
        sl = max(s_n // args.steps, 1)
        kind, splits = knn.last_select_kernel()
        kname = {"warp per row": "select_warp_kernel", "cluster per row": "select_cluster_kernel",
                 "two-pass warp per row": "select_warp2p_kernel"}.get(kind, "select_ring_kernel")
        rooflines.append((s_ms, hbm_roof(f"{kname} (a-S4, {kind})", kname, s_ms, s_n,
                                         rows_w / sl * (cols_w * 4.0 + k * 8.0))))
    if m_n and pivot_plan:
        cands = knn.last_candidates()  # survivors of the partition (whole call)
        sel_rows = R_local if sym_shard else rows_w
        cs_name = ("candidate_recompute_kernel" if pivot1 else "candidate_select_kernel") if k <= 32 \
            else "candidate_select_warp_kernel"
        if pivot1:
            # the re-evaluation gathers the fp32 rows of its ~40 survivors per row from L2: its
            # roofline is the measured L2 gather rate of that pattern (tools/l2_gather_probe.cu,
            # profiles/l2_gather_probe.json); |R| from one untimed call with the library's
            # counter (KNN_RECOMP_STATS counts the re-evaluated set instead of the lists)
            os.environ["KNN_RECOMP_STATS"] = "1"
            step()
            torch.cuda.synchronize()
            reev = knn.last_candidates()
            del os.environ["KNN_RECOMP_STATS"]
            step()  # (restores the library's candidate count of a normal call)
            torch.cuda.synchronize()
            try:
                with open(os.path.join(ROOT, "profiles", "l2_gather_probe.json")) as f:
                    l2peak = json.load(f)["l2_gather_gbs"]
            except Exception:
                l2peak = None
            r = hbm_roof(f"{cs_name} (exact select of the partition: fp32 re-evaluation of the survivors "
                         f"near the k-th, rows gathered from L2)", cs_name, m_ms, m_n,
                         reev * d * 4.0 + cands * 8.0 + sel_rows * (4.0 + k * 8.0))
            if l2peak:
                r.update({"bound": "l2", "peak": l2peak, "frac": r["achieved"] / l2peak,
                          "peak_kind": "measured L2 gather rate, random 1 KB rows of a 64 MB L2-resident "
                                       "matrix (profiles/l2_gather_probe.json)"})
            r["reevaluated_per_row"] = reev / max(sel_rows, 1)
            rooflines.append((m_ms, r))
        else:
            rooflines.append((m_ms, hbm_roof(f"{cs_name} (exact select of the partition)",
                                             cs_name, m_ms, m_n,
                                             cands * 8.0 + sel_rows * (4.0 + k * 8.0))))
        rooflines[-1][1]["candidates_per_row"] = cands / max(sel_rows, 1)
    if x_n:  # Par-2: the k-way merge of the ranks' partial lists of this rank's rows
        rooflines.append((x_ms, hbm_roof("merge_lists_kernel (a-S6, corpus-sharded k-way merge)",
                                         "merge_lists_kernel", x_ms, x_n, R_local * k * 8.0 * (world + 1))))
    rooflines.sort(key=lambda x: -x[0])
    roofline = dict(rooflines[0][1])
    roofline["others"] = [r for _, r in rooflines[1:]]
    roofline["step_share"] = {"partition": f_ms / total_ms, "gemm": g_ms / total_ms,
                              "select": s_ms / total_ms, "candidate_select": m_ms / total_ms,
                              "prep": p_ms / total_ms, "shard_merge": x_ms / total_ms}
    if roofline["bound"] == "tensor":
        # the step against the dominant kernel's own floor (its flop at the burst peak)
        roofline["step_floor_frac"] = roofline["flop_per_launch"] * (roofline["launches"] / args.steps) / \
            (roofline["peak"] * 1e12) / (ms_per_step * 1e-3)
    roofline["plan"] = {0: "blocked distances + select",
                        2: "symmetric k-NNG distances (PAPER.md:83 transpose reuse) + select",
                        3: "pivot (quickselect partition, PAPER.md:56) over the symmetric GEMM",
                        4: "pivot (quickselect partition, PAPER.md:56) over the GEMM",
                        5: "pivot (quickselect partition, PAPER.md:56) over the symmetric single-product GEMM, "
                           "survivors re-evaluated in fp32",
                        6: "pivot (quickselect partition, PAPER.md:56) over the single-product GEMM, "
                           "survivors re-evaluated in fp32"}.get(
                            plan_code, "unknown")

    # ---- e2e: the public host-buffer API, H2D of the inputs and D2H of the results inside
    e2e = None
    if not args.no_e2e:
        lo, hi = sharded.block_range(M, world, rank)
        Xh = torch.empty((N, d), dtype=torch.float32, pin_memory=True)
        if rank == 0:
            Xh.copy_(torch.from_numpy(X_host))
        else:
            Xh.copy_(X.cpu())
        Xn = Xh.numpy()
        oi = torch.empty((hi - lo, k), dtype=torch.int32, pin_memory=True).numpy()
        od = torch.empty((hi - lo, k), dtype=torch.float32, pin_memory=True).numpy()
        if search:
            Qh = torch.empty((hi - lo, d), dtype=torch.float32, pin_memory=True)
            Qh.copy_(torch.from_numpy(Q_host[lo:hi]) if rank == 0 else Q[lo:hi].cpu())
            Qn = Qh.numpy()
        else:
            Qn = Xn[lo:hi]

        def e2e_step():
            knn.search_block_host(Qn, Xn, k, self_shift=knn.NO_SELF if search else lo, out=(oi, od))

        for _ in range(2):
            e2e_step()
        e_ms = 0.0
        for _ in range(max(3, args.steps // 2)):
            flush.zero_()
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()
            e_ms += (time.perf_counter() - t0) * 1e3
            barrier()
        e_ms /= max(3, args.steps // 2)
        te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": M / (float(te.item()) / 1e3), "unit": "points/s",
               "h2d_bytes_per_step": int((N + (hi - lo if search else 0)) * d * 4),
               "d2h_bytes_per_step": int((hi - lo) * k * 8),
               "api": "knn_search_block_host (pinned host buffers)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        threads = oracle.default_threads()
        rps, R, dt = oracle_rows_per_s(X_host, k, not search, args.cpu_seconds, threads,
                                       Q=Q_host if search else None)
        cpu = {"value": rps, "unit": "points/s", "cores": threads, "kind": "oracle",
               "sample": f"{R} seeded query rows of the {workload_name(cfg)} ({dt:.1f} s; fp64 direct "
                         f"distances + full std::sort per row)"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(cfg), "N": N, "M": M, "d": d, "k": k,
                       "sharding": {"sym": "upper triangle split over the ranks (Par-3): bcast X, pivots "
                                            "all-gathered, partition GEMM on 1/G of the 256x256 blocks, select "
                                            "reading the ranks' candidate lists in peer memory, all-gather",
                                    "corpus": "corpus columns (Par-2): bcast X, per-rank partial top-k of all rows, "
                                              "all-to-all of row blocks, k-way merge kernel, all-gather",
                                    "query": "query rows (Par-1): bcast X, per-rank rows, all-gather"}[shard_ran]
                                   if world > 1 else f"one GPU ({shard_ran} call as one rank)",
                       "collectives": ("NCCL inside libknn (knn_comm_init)" if not share else
                                       "host transport (ranks share one GPU; not a reported number)")
                                      if world > 1 else "none",
                       "gemm": "tcgen05 3-pass split-fp16 (FP32-accurate), fp32 accumulate",
                       "l2": "flushed before every timed step (256 MiB write, untimed)"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches,
            "plan": roofline["plan"],
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def self_launch(args):
    """--gpus N > 1 without a launcher: start N ranks (one per GPU) with torch.distributed.run
    on 127.0.0.1 and relay their output (rank 0 prints the JSON line)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
