#!/usr/bin/env python
"""NEXT-4 measurement: out-of-core k-NN (knn_search_streamed) vs the device-resident call.

Workload: M queries, N corpus points, d, k (default 65536 x 2^21 x 256, k = 32; uniform
fp32, datagen seeds).  Both inputs live in host memory for the streamed call; the corpus
is streamed in chunks of --chunk points with copy/compute overlap.  Reported: wall time
of the blocking streamed call (host arrays in, host results out), the device-resident
time of knn_search on the same inputs already in HBM (kernel-only reference), the H2D
bytes moved and the overlap efficiency resident / streamed.  Results are compared bit
for bit.

  python scripts/stream_bench.py [--M 65536 --N 2097152 --d 256 --k 32 --chunk 262144]
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

from paper_1309_5478_b200 import datagen, knn  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=65536)
    ap.add_argument("--N", type=int, default=1 << 21)
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--chunk", type=int, default=262144)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "stream_bench.json"))
    a = ap.parse_args()
    Q = datagen.points(a.M, a.d, "uniform", seed=1309200)
    X = datagen.points(a.N, a.d, "uniform", seed=1309201)
    Qp = torch.from_numpy(Q).pin_memory()
    Xp = torch.from_numpy(X).pin_memory()
    res = {"M": a.M, "N": a.N, "d": a.d, "k": a.k, "chunk": a.chunk}
    for name, (qa, xa) in {"pinned": (Qp.numpy(), Xp.numpy()), "pageable": (Q, X)}.items():
        knn.search_streamed(qa, xa, a.k, chunk_points=a.chunk)  # warm-up
        t = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            out = knn.search_streamed(qa, xa, a.k, chunk_points=a.chunk)
            t.append(time.perf_counter() - t0)
        res[name + "_s"] = min(t)
        res[name + "_queries_per_s"] = a.M / min(t)
    Qd, Xd = Qp.cuda(), Xp.cuda()
    knn.search(Qd, Xd, a.k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        ri, rd = knn.search(Qd, Xd, a.k)
    e1.record()
    torch.cuda.synchronize()
    res["resident_s"] = e0.elapsed_time(e1) / 1e3 / a.reps
    res["h2d_bytes"] = (a.M + a.N) * a.d * 4
    res["d2h_bytes"] = a.M * a.k * 8
    res["overlap_efficiency_pinned"] = res["resident_s"] / res["pinned_s"]
    res["bit_identical"] = bool(np.array_equal(out[0], ri.cpu().numpy()) and
                                np.array_equal(out[1].view(np.uint32), rd.cpu().numpy().view(np.uint32)))
    res["h2d_gbs_pinned"] = res["h2d_bytes"] / res["pinned_s"] / 1e9
    print(json.dumps(res), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
