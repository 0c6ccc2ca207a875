"""Multi-GPU drivers: one process per GPU, torch.distributed (NCCL) for the plumbing.

Two shardings of the brute-force k-NN (the paper is single-GPU and names
"batch execution with data partitioning ... merging of results" as future work,
PAPER.md:102):

* ``graph_query_sharded`` (Par-1): query rows are independent.  Rank 0's dataset is
  broadcast once over NVLink, each rank runs the whole hot path (norms -> GEMM ->
  select) on its contiguous block of ceil(N/G) query rows against all N points, and the
  M×k results are all-gathered.  The only exchanges are the input broadcast and the
  output gather; there is no collective inside the hot path.
* ``graph_sym_sharded`` (Par-3, the default k-NNG path for N >= 16384): the ranks split
  the UPPER TRIANGLE of the distance matrix (the transpose reuse of PAPER.md:83 survives
  sharding; a row split would double each rank's multiply work): every rank computes the
  pivots of its row block (the pivot plan's sample pass), the pivots are all-gathered,
  every rank runs the partition GEMM over 1/G of the triangle's 256x256 blocks appending
  candidates of ANY row to its own lists, and each rank's select kernel reads the G ranks'
  lists of its row block straight from their memory (CUDA IPC over NVLink) before the
  results are all-gathered.  Bit-identical to one GPU.
* ``graph_corpus_sharded`` (Par-2): corpus columns are split in G contiguous blocks;
  every rank computes partial top-k lists of ALL rows against its block (global self
  exclusion and global indices via knn_search_block's self_shift / idx_offset), an
  all-to-all hands each rank the G partial lists of its own row block, the k-way merge
  kernel (knn_merge) produces its final rows, and an all-gather assembles the graph.
  Equal to the unsharded graph bit-for-bit: (distance, index) is a total order and the
  shards are contiguous index ranges.

The per-rank compute is injected (``compute`` / ``merge``) so the same orchestration is
exercised by the world-size-2 gloo tests on CPU with oracle stand-ins; by default it is
the CUDA library (there is no CPU fallback in the product path).
"""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist


def block_range(n: int, parts: int, r: int):
    """Contiguous block r of ceil(n/parts)-sized blocks of range(n): [lo, hi)."""
    per = -(-n // parts)
    lo = min(n, r * per)
    return lo, min(n, lo + per)


def _default_compute(Q, X, k, metric, self_shift, idx_offset):
    from . import knn
    return knn.search_block(Q, X, k, metric=metric, self_shift=self_shift, idx_offset=idx_offset)


def _default_merge(part_dist, part_idx, offsets):
    from . import knn
    return knn.merge(part_dist, part_idx, offsets)


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def broadcast_points(X, group=None, src=0):
    """Broadcast rank `src`'s N×d point set (in place on every rank)."""
    dist.broadcast(X, src=src, group=group)
    return X


def graph_query_sharded(X, k, metric=0, group=None, compute=None, broadcast=True):
    """k-NNG of X with the query rows sharded over the ranks of `group` (Par-1).

    X: N×d fp32 tensor on this rank's device, valid on rank 0 (broadcast here unless
    broadcast=False).  Returns the full (idx N×k int32, dist N×k fp32) on every rank."""
    compute = compute or _default_compute
    G, r = _world(group)
    N = X.shape[0]
    if broadcast and G > 1:
        broadcast_points(X, group)
    if G == 1:
        return compute(X, X, k, metric, 0, 0)
    per = -(-N // G)
    lo, hi = block_range(N, G, r)
    out_i = torch.zeros((per, k), dtype=torch.int32, device=X.device)
    out_d = torch.full((per, k), float("inf"), dtype=torch.float32, device=X.device)
    if hi > lo:
        i, d = compute(X[lo:hi], X, k, metric, lo, 0)  # self pair: column lo + i
        out_i[: hi - lo] = i
        out_d[: hi - lo] = d
    all_i = torch.empty((G * per, k), dtype=torch.int32, device=X.device)
    all_d = torch.empty((G * per, k), dtype=torch.float32, device=X.device)
    dist.all_gather_into_tensor(all_i, out_i, group=group)
    dist.all_gather_into_tensor(all_d, out_d, group=group)
    return all_i[:N], all_d[:N]


def search_query_sharded(Q, X, k, group=None, compute=None, broadcast=True):
    """k-NN search with the query rows sharded (Par-1); Q and X valid on rank 0."""
    compute = compute or _default_compute
    G, r = _world(group)
    M = Q.shape[0]
    if broadcast and G > 1:
        broadcast_points(X, group)
        broadcast_points(Q, group)
    per = -(-M // G)
    lo, hi = block_range(M, G, r)
    out_i = torch.zeros((per, k), dtype=torch.int32, device=X.device)
    out_d = torch.full((per, k), float("inf"), dtype=torch.float32, device=X.device)
    if hi > lo:
        i, d = compute(Q[lo:hi], X, k, 0, -(2 ** 63), 0)
        out_i[: hi - lo] = i
        out_d[: hi - lo] = d
    if G == 1:
        return out_i[:M], out_d[:M]
    all_i = torch.empty((G * per, k), dtype=torch.int32, device=X.device)
    all_d = torch.empty((G * per, k), dtype=torch.float32, device=X.device)
    dist.all_gather_into_tensor(all_i, out_i, group=group)
    dist.all_gather_into_tensor(all_d, out_d, group=group)
    return all_i[:M], all_d[:M]


def _all_gather_rows(t, G, group):
    """all_gather_into_tensor of equal row blocks; staged through host memory when the
    backend cannot gather device tensors (gloo, used by the one-GPU tests)."""
    out = torch.empty((G * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    if t.is_cuda and dist.get_backend(group) != "nccl":
        host = torch.empty(out.shape, dtype=t.dtype)
        dist.all_gather_into_tensor(host, t.cpu(), group=group)
        out.copy_(host)
    else:
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    return out


def peer_merge(part_i, part_d, k, row0, rows, group=None):
    """Fused exchange + merge of the corpus-sharded k-NNG (SURVEY §8(e) "better Par-2"):
    every rank maps its peers' partial-list buffers (CUDA IPC; over NVLink between GPUs)
    and the merge kernel reads the G lists of its own row block [row0, row0 + rows)
    straight from peer memory — no all-to-all copy of the lists.  The partial lists must be
    complete on every rank before any rank reads them (synchronize + barrier), and stay
    alive until every rank has finished reading (second barrier)."""
    from . import knn
    G, r = _world(group)
    hi, oi = knn.ipc_export(part_i)
    hd, od = knn.ipc_export(part_d)
    table = [None] * G
    dist.all_gather_object(table, (hi, oi, hd, od), group=group)
    dptrs, iptrs = [], []
    for g, (h_i, o_i, h_d, o_d) in enumerate(table):
        if g == r:
            dptrs.append(part_d.data_ptr())
            iptrs.append(part_i.data_ptr())
        else:
            dptrs.append(knn.ipc_open(h_d, o_d, part_d.device.index))
            iptrs.append(knn.ipc_open(h_i, o_i, part_i.device.index))
    torch.cuda.synchronize(part_i.device)
    dist.barrier(group=group)
    mi, md = knn.merge_lists(dptrs, iptrs, row0, rows, k, device=part_i.device.index)
    torch.cuda.synchronize(part_i.device)
    dist.barrier(group=group)
    knn.ipc_close_all(part_i.device.index)
    return mi, md


class _SymLists:
    """Per-process candidate lists of the symmetric sharded k-NNG, kept across calls so
    that their CUDA IPC mappings are exported / opened once."""
    cache = {}

    @classmethod
    def get(cls, N, cap, device, group):
        key = (N, cap, device.index, id(group))
        ent = cls.cache.get(key)
        if ent is None:
            cnt = torch.zeros(N, dtype=torch.int32, device=device)
            ckey = torch.empty((N, cap), dtype=torch.int32, device=device)
            cidx = torch.empty((N, cap), dtype=torch.int32, device=device)
            ent = {"cnt": cnt, "ckey": ckey, "cidx": cidx, "ptrs": None}
            cls.cache[key] = ent
        return ent


def _agree(ok, device, group):
    """True on every rank iff `ok` holds on every rank (one MAX all-reduce)."""
    nccl = dist.get_backend(group) == "nccl"
    f = torch.tensor([0 if ok else 1], dtype=torch.int32, device=device if nccl else "cpu")
    dist.all_reduce(f, op=dist.ReduceOp.MAX, group=group)
    return int(f.item()) == 0


def _peer_pointers(ent, group):
    """Device pointers of every rank's (cnt, ckey, cidx): own ones local, peers' mapped
    with CUDA IPC (exchanged once with all_gather_object).  None on every rank if any rank
    could not export or map (e.g. an allocator without IPC support): the caller falls back
    to a path without peer mappings."""
    from . import knn
    if ent["ptrs"] is not None:
        return ent["ptrs"] if ent["ptrs"] != "none" else None
    G, r = _world(group)
    try:
        if os.environ.get("KNN_SHARD_NO_IPC", "0") == "1":  # tests: force the fallback
            raise RuntimeError("CUDA IPC disabled")
        mine = tuple(knn.ipc_export(ent[n]) for n in ("cnt", "ckey", "cidx"))
    except Exception:
        mine = None
    table = [None] * G
    dist.all_gather_object(table, mine, group=group)
    dev = ent["cnt"].device.index
    ptrs = ([], [], [])
    ok = all(t is not None for t in table)
    if ok:
        try:
            for g in range(G):
                for j, name in enumerate(("cnt", "ckey", "cidx")):
                    if g == r:
                        ptrs[j].append(ent[name].data_ptr())
                    else:
                        h, off = table[g][j]
                        ptrs[j].append(knn.ipc_open(h, off, dev))
        except Exception:
            ok = False
    if not _agree(ok, ent["cnt"].device, group):
        ent["ptrs"] = "none"
        return None
    ent["ptrs"] = ptrs
    return ptrs


def graph_sym_sharded(X, k, metric=0, group=None, broadcast=True):
    """k-NNG of X with the upper triangle of the distance matrix split over the ranks
    (Par-3).  X: N x d fp32 on this rank's device, valid on rank 0 (broadcast here unless
    broadcast=False).  Returns the full (idx N x k, dist N x k) on every rank.  Falls back
    to the query-row sharding (Par-1, materialised plan) if any rank's certificate fails."""
    from . import knn
    G, r = _world(group)
    N, d = X.shape
    if broadcast and G > 1:
        broadcast_points(X, group)
    per = -(-N // G)
    lo, hi = block_range(N, G, r)
    npad = -(-N // 256) * 256
    thr = torch.full((max(npad, G * per),), float("nan"), dtype=torch.float32, device=X.device)
    if hi > lo:
        knn.graph_pivots(X, k, lo, hi - lo, thr, metric=metric)
    if G > 1:
        blk = thr[r * per:(r + 1) * per].clone()
        gathered = torch.empty(G * per, dtype=torch.float32, device=X.device)
        if X.is_cuda and dist.get_backend(group) != "nccl":
            host = torch.empty(G * per, dtype=torch.float32)
            dist.all_gather_into_tensor(host, blk.cpu(), group=group)
            gathered.copy_(host)
        else:
            dist.all_gather_into_tensor(gathered, blk, group=group)
        thr[:G * per] = gathered
        thr[N:] = float("nan")
    units = knn.graph_units(N)
    u_lo, u_hi = block_range(units, G, r)
    cap = knn.graph_list_cap(k)
    ent = _SymLists.get(N, cap, X.device, group)
    knn.graph_partition(X, k, thr, u_lo, u_hi, ent["cnt"], ent["ckey"], ent["cidx"], metric=metric)
    if G > 1:
        ptrs = _peer_pointers(ent, group)
        if ptrs is None:  # no CUDA IPC between these ranks: shard query rows instead
            return graph_query_sharded(X, k, metric=metric, group=group, broadcast=False)
        # every rank's partition must be complete before any rank reads its lists: with NCCL a
        # stream-ordered all-reduce is that barrier on the device (no host synchronisation);
        # host-side backends synchronise explicitly
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(torch.zeros(1, dtype=torch.int32, device=X.device), group=group)
        else:
            torch.cuda.synchronize(X.device)
            dist.barrier(group=group)
    else:
        ptrs = ([ent["cnt"].data_ptr()], [ent["ckey"].data_ptr()], [ent["cidx"].data_ptr()])
    ok = True
    out_i = torch.zeros((per, k), dtype=torch.int32, device=X.device)
    out_d = torch.full((per, k), float("inf"), dtype=torch.float32, device=X.device)
    if hi > lo:
        try:
            i, dd = knn.graph_gather_select(ptrs[0], ptrs[1], ptrs[2], cap, N, k, lo, hi - lo,
                                            device=X.device.index)
            out_i[: hi - lo] = i
            out_d[: hi - lo] = dd
        except knn.KnnError as e:
            if e.status != 7:  # KNN_ERR_INTERNAL: certificate / overflow
                raise
            ok = False
    if G == 1:
        if not ok:
            return graph_query_sharded(X, k, metric=metric, group=group, broadcast=False)
        return out_i[:N], out_d[:N]
    # any rank's certificate failed?  (every rank calls this after its select returned, so
    # when it completes no rank still reads another's lists)
    all_ok = _agree(ok, X.device, group)
    if dist.get_backend(group) != "nccl":
        dist.barrier(group=group)
    if not all_ok:
        return graph_query_sharded(X, k, metric=metric, group=group, broadcast=False)
    all_i = _all_gather_rows(out_i, G, group)
    all_d = _all_gather_rows(out_d, G, group)
    return all_i[:N], all_d[:N]


def graph_corpus_sharded(X, k, metric=0, group=None, compute=None, merge=None, broadcast=True,
                         exchange="all_to_all", peer_merge_fn=None):
    """k-NNG of X with the corpus columns sharded over the ranks (Par-2).

    exchange="all_to_all": an all-to-all hands each rank the G partial lists of its row
    block, merged with knn_merge.  exchange="peer": each rank merges its row block straight
    from its peers' partial lists mapped over CUDA IPC (peer_merge).  Needs k <= the
    smallest column block.  Returns the full graph on every rank."""
    compute = compute or _default_compute
    merge = merge or _default_merge
    G, r = _world(group)
    N = X.shape[0]
    if broadcast and G > 1:
        broadcast_points(X, group)
    c0, c1 = block_range(N, G, r)
    if min(block_range(N, G, g)[1] - block_range(N, G, g)[0] for g in range(G)) < k:
        raise ValueError("corpus sharding needs k <= N/G")
    per = -(-N // G)
    # partial lists of every row against columns [c0, c1), rows padded to G*per
    part_i = torch.zeros((G * per, k), dtype=torch.int32, device=X.device)
    part_d = torch.full((G * per, k), float("inf"), dtype=torch.float32, device=X.device)
    i, d = compute(X, X[c0:c1], k, metric, -c0, c0)  # self: global column c0 + j == row i
    part_i[:N] = i
    part_d[:N] = d
    if G == 1:
        return merge(part_d[None, :N], part_i[None, :N], np.zeros(1, np.int64))
    if exchange == "peer":
        mi, md = (peer_merge_fn or peer_merge)(part_i, part_d, k, r * per, per, group)
    else:
        # all-to-all: rank g receives, from every rank, the partial lists of rows block g
        recv_i = torch.empty_like(part_i)
        recv_d = torch.empty_like(part_d)
        dist.all_to_all_single(recv_i, part_i, group=group)
        dist.all_to_all_single(recv_d, part_d, group=group)
        # recv[s*per:(s+1)*per] = rank s's lists for this rank's rows -> [G][per][k]
        mi, md = merge(recv_d.view(G, per, k), recv_i.view(G, per, k), np.zeros(G, np.int64))
    all_i = _all_gather_rows(mi.contiguous(), G, group)
    all_d = _all_gather_rows(md.contiguous(), G, group)
    return all_i[:N], all_d[:N]
