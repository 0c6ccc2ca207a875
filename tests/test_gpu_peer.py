"""knn_merge_lists (the merge over a table of list pointers, local or peer-mapped with
knn_ipc_open) must equal knn_merge; knn_ipc_* round trip within one process."""
import numpy as np
import pytest

from paper_1309_5478_b200 import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def knn():
    from paper_1309_5478_b200 import knn as k
    return k


def test_merge_lists_equals_merge():
    g = np.random.Generator(np.random.Philox(5))
    G, M, k = 5, 700, 40
    pd = np.sort(g.random((G, M + 30, k), dtype=np.float32), axis=2)
    pi = g.integers(0, 1 << 20, size=(G, M + 30, k)).astype(np.int32)
    offs = np.arange(G, dtype=np.int64) * 1000
    row0 = 30
    tens_d = [torch.from_numpy(pd[gg]).cuda() for gg in range(G)]   # separate allocations
    tens_i = [torch.from_numpy(pi[gg]).cuda() for gg in range(G)]
    got = knn().merge_lists([t.data_ptr() for t in tens_d], [t.data_ptr() for t in tens_i],
                            row0, M, k, offs)
    ref = knn().merge(torch.from_numpy(np.ascontiguousarray(pd[:, row0:])).cuda(),
                      torch.from_numpy(np.ascontiguousarray(pi[:, row0:])).cuda(), offs)
    assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1])


def test_ipc_export_open_roundtrip():
    kn = knn()
    t = torch.arange(1000, dtype=torch.int32, device="cuda")
    sub = t[100:]
    h, off = kn.ipc_export(sub)
    assert len(h) == 64 and off >= 400
    kn.ipc_close_all()
