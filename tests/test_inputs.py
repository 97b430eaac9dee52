"""The seeded input generators: determinism and numpy/torch bit-equality (CPU)."""
import numpy as np
import pytest
import torch

from inputs import graphs, rng


def test_hash_numpy_equals_torch():
    idx = np.arange(0, 5000, 7, dtype=np.uint64)
    for seed, stream in [(0, 0), (1, 100), (2**40 + 3, 401)]:
        a = rng.counter_hash_np(seed, stream, idx)
        b = rng.counter_hash_torch(seed, stream, torch.from_numpy(idx.astype(np.int64))).numpy().view(np.uint64)
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("kw", [dict(kind="rmat", seed=1, scale=10),
                                dict(kind="rmat", seed=3, scale=11, permute=True),
                                dict(kind="er", seed=2, n=3000, m_raw=40000),
                                dict(kind="rmat", seed=5, scale=10, permute=True, values=True, transpose=True)])
def test_graph_numpy_equals_torch_cpu(kw):
    kind = kw.pop("kind")
    a = graphs.make_graph(kind, **kw)
    b = graphs.make_graph(kind, backend="torch", device="cpu", **kw).to_numpy()
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.col, b.col)
    if a.values is not None:
        np.testing.assert_array_equal(a.values, b.values)


def test_csr_canonical_and_config_shapes():
    g = graphs.make_config("c1")
    assert g.n_src == 1024 and 11000 < g.m < 13000          # ~16K raw edges, ~25% duplicates
    for u in range(g.n_src):
        row = g.col[g.row_ptr[u]:g.row_ptr[u + 1]].astype(np.int64)
        assert np.all(np.diff(row) > 0)
    # unpermuted RMAT: low IDs are hubs (BASELINE config 1 has no relabelling)
    deg = np.diff(g.row_ptr)
    assert deg[:256].sum() > 0.45 * g.m
    # determinism
    g2 = graphs.make_config("c1")
    np.testing.assert_array_equal(g.col, g2.col)


def test_values_exact_in_unit_interval():
    v = graphs.make_x(100000, 5)
    assert v.dtype == np.float32 and v.min() >= -1 and v.max() < 1
    assert abs(float(v.mean())) < 0.01


def _bfs_python(n, row_ptr, col):
    """Reading R16 written out with Python lists (small graphs only)."""
    deg = [int(row_ptr[u + 1] - row_ptr[u]) for u in range(n)]
    order = sorted(range(n), key=lambda u: (-deg[u], u))
    new = [-1] * n
    nxt = 0
    for s in order:
        if new[s] >= 0:
            continue
        new[s] = nxt
        nxt += 1
        q = [s]
        while q:
            u = q.pop(0)
            for v in col[row_ptr[u]:row_ptr[u + 1]]:
                if new[v] < 0:
                    new[v] = nxt
                    nxt += 1
                    q.append(int(v))
    return new


def test_bfs_order_matches_python_bfs_and_relabels_isomorphically():
    import numpy as np
    from inputs import graphs
    for seed, scale in ((1, 8), (2, 10)):
        g = graphs.make_graph("rmat", seed, scale=scale, permute=True)
        nid = graphs.bfs_order(g.n_src, g.row_ptr, g.col)
        assert nid.tolist() == _bfs_python(g.n_src, g.row_ptr, g.col)
        assert sorted(nid.tolist()) == list(range(g.n_src))
        h = graphs.relabel(g, nid)
        assert h.m == g.m
        rows = np.repeat(np.arange(g.n_src), np.diff(g.row_ptr))
        old = set(zip(nid[rows].tolist(), nid[g.col.astype(np.int64)].tolist()))
        rows2 = np.repeat(np.arange(h.n_src), np.diff(h.row_ptr))
        assert old == set(zip(rows2.tolist(), h.col.astype(np.int64).tolist()))
    # the start vertex (max out-degree) gets label 0
    deg = np.diff(g.row_ptr)
    assert nid[int(np.argmax(deg))] == 0


def test_relabel_torch_equals_numpy():
    import numpy as np
    import torch
    from inputs import graphs
    g = graphs.make_graph("rmat", 3, scale=9, permute=True)
    nid = graphs.bfs_order(g.n_src, g.row_ptr, g.col)
    a = graphs.relabel(g, nid)
    gt = graphs.GraphCSR("t", g.n_src, g.n_dst, torch.from_numpy(g.row_ptr),
                         torch.from_numpy(g.col.view(np.int32)), None, {})
    b = graphs.relabel(gt, torch.from_numpy(nid)).to_numpy()
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.col, b.col)


def test_column_prefix_keeps_each_rows_leading_columns():
    g = graphs.make_graph("rmat", 5, scale=10, permute=True, values=True, transpose=True)
    h = graphs.column_prefix(g, 300)
    assert (h.n_src, h.n_dst) == (g.n_src, 300) and h.m == int((g.col < 300).sum())
    for u in range(0, g.n_src, 7):
        a = g.col[g.row_ptr[u]:g.row_ptr[u + 1]]
        va = g.values[g.row_ptr[u]:g.row_ptr[u + 1]]
        np.testing.assert_array_equal(h.col[h.row_ptr[u]:h.row_ptr[u + 1]], a[a < 300])
        np.testing.assert_array_equal(h.values[h.row_ptr[u]:h.row_ptr[u + 1]], va[a < 300])
    ht = graphs.column_prefix(graphs.make_graph("rmat", 5, scale=10, permute=True, values=True, transpose=True,
                                                backend="torch"), 300).to_numpy()
    np.testing.assert_array_equal(ht.row_ptr, h.row_ptr)
    np.testing.assert_array_equal(ht.col, h.col)
    np.testing.assert_array_equal(ht.values, h.values)
