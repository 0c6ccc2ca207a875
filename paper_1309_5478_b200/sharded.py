"""Multi-GPU plumbing: one process per GPU; torch.distributed only starts the communicator.

The shardings themselves live in libknn (include/knn.h "multi-GPU", csrc/shard.cu):
``knn_graph_sharded`` / ``knn_search_sharded`` broadcast the points, run the per-rank
hot path, exchange partial results and all-gather the lists, with the collectives issued
by the library on the caller's stream ("batch execution with
data partitioning ... merging of results"):

* ``query``  (Par-1): query rows split; each rank runs the whole path on its rows.
* ``corpus`` (Par-2): corpus columns split; per-rank partial top-k of every row, an
  all-to-all of the row blocks, the k-way merge kernel, all-gather (C5's layout).
* ``sym``    (Par-3, k-NNG): the ranks split the upper triangle of the distance matrix
  (PAPER.md:83's transpose reuse survives sharding); the select reads every rank's
  candidate lists in peer memory over NVLink (CUDA IPC mappings exchanged once).

This module only creates the communicator: for an NCCL process group it ships an NCCL
unique id made by rank 0 (``knn_comm_unique_id`` / ``knn_comm_init``); for any other
backend (gloo: tests with several ranks sharing one GPU, which NCCL refuses) it hands the
library a host transport (``knn_comm_init_ops``) whose four collectives are the process
group's, on numpy views of the library's pinned staging buffers.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import knn


def block_range(n: int, parts: int, r: int):
    """Contiguous block r of ceil(n/parts)-sized blocks of range(n): [lo, hi) — the
    library's own split (knn_shard_range)."""
    return knn.shard_range(n, parts, r)


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


class TorchHostTransport:
    """knn_comm_ops over a torch.distributed process group, on host (numpy) buffers.
    Marshalling only: each method is one collective of the group."""

    def __init__(self, group=None):
        self.group = group
        self.G, self.rank = _world(group)

    def allgather(self, send, recv):
        n = send.shape[0]
        out = [torch.from_numpy(recv[g * n:(g + 1) * n]) for g in range(self.G)]
        dist.all_gather(out, torch.from_numpy(send), group=self.group)

    def broadcast(self, buf, root):
        src = dist.get_global_rank(self.group, root) if self.group is not None else root
        dist.broadcast(torch.from_numpy(buf), src=src, group=self.group)

    def alltoall(self, send, recv):
        dist.all_to_all_single(torch.from_numpy(recv), torch.from_numpy(send), group=self.group)

    def allreduce_max(self, buf):
        t = torch.from_numpy(buf)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)


def init(group=None, device=None, transport="auto"):
    """Create the library's communicator for this rank (collective over `group`).

    transport: "nccl" (NCCL over NVLink; the default for an NCCL process group), "host"
    (the group's own collectives through pinned host staging; the default otherwise)."""
    G, r = _world(group)
    nccl = transport == "nccl" or (transport == "auto" and G > 1 and dist.get_backend(group) == "nccl")
    if G == 1 and transport != "nccl":
        knn.comm_destroy(device)
        return
    if nccl:
        obj = [knn.comm_unique_id() if r == 0 else None]
        if G > 1:
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(obj, src=src, group=group)
        knn.comm_init(r, G, obj[0], device)
    else:
        knn.comm_init_ops(r, G, TorchHostTransport(group), device)


def graph(X, k, mode="sym", metric=0, out=None):
    """k-NNG of X over the ranks (knn_graph_sharded): X valid on rank 0 (broadcast into X
    on the others); the full (idx N×k, dist N×k) on every rank."""
    return knn.graph_sharded(X, k, mode=mode, metric=metric, out=out)


def search(Q, X, k, mode="query", out=None):
    """k-NN search over the ranks (knn_search_sharded): Q, X valid on rank 0."""
    return knn.search_sharded(Q, X, k, mode=mode, out=out)
