"""Parity of the CUDA path (through the C ABI) against the fp64 CPU oracle.

* layout (a0): bit-exact, every array, on fixtures, random graphs and edge cases;
* scatter (a1): bit-exact given the same fp32 input;
* PageRank (a1-a4): max relative error <= 1e-5 per vertex and L1 <= 1e-6 after
  the stated iterations (BASELINE.json north_star), plus bit-reproducibility;
* SpMV (a5): |y - y_oracle| <= 1e-5 * sum|a x| + deg * 2^-F (R19).
"""
import json
import os

import numpy as np
import pytest

import oracle
from inputs import graphs
from tests.gpu_util import d2h, spmv_fbits, to_device

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def pcpm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1709_07122_b200 import pcpm as p
    return p


def build(p, g, b, flags=0, device=True):
    if device:
        rp, col, val = to_device(g)
        keep = (rp, col, val)
    else:
        rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(g.col, dtype=np.uint32)
        val = None if g.values is None else np.ascontiguousarray(g.values, dtype=np.float32)
        keep = (rp, col, val)
    csr = p.make_csr(g.n_src, g.n_dst, rp, col, val)
    h = p.pcpm_build_ex(csr, b, flags, None)
    del keep
    return h


def export(p, h):
    info = p.pcpm_get_info(h)
    v = p.pcpm_export_layout(h)
    m, ep, ks, kd = info.nnz, info.e_prime, info.k_src, info.k_dst
    out = dict(
        info=info,
        ids=d2h(v.ids, m, np.uint32) if v.ids else None,
        png_src=d2h(v.png_src, ep, np.uint32) if v.png_src else None,
        ids16=d2h(v.ids16, m, np.uint16),
        png_src16=d2h(v.png_src16, ep, np.uint16),
        png_off=d2h(v.png_off, ks * (kd + 1), np.uint32).reshape(ks, kd + 1),
        upd_off=d2h(v.upd_off, ks * kd, np.uint32).reshape(ks, kd),
        bin_id_start=d2h(v.bin_id_start, kd + 1, np.uint32),
        bin_upd_start=d2h(v.bin_upd_start, kd + 1, np.uint32),
        chunk_base=d2h(v.chunk_base, (m + 2047) // 2048 * 16 + 1, np.uint32),
        out_degree=d2h(v.out_degree, info.n_src, np.uint32),
        w=d2h(v.w, m, np.float32) if v.w else None,
        view=v,
    )
    return out


def assert_layout_equal(g, lay_gpu, b, compress=True):
    if compress:
        ref = oracle.layout(g.n_src, g.n_dst, g.row_ptr, g.col, b, val=g.values)
        ids = ref.ids
    else:
        ref = oracle.layout(g.n_src, g.n_dst, g.row_ptr, g.col, b, val=g.values)
        ids = None
    info = lay_gpu["info"]
    assert info.k_src == ref.k_src and info.k_dst == ref.k_dst
    qmask = np.uint32((1 << b) - 1)
    if compress:
        assert info.e_prime == ref.e_prime
        if lay_gpu["ids"] is not None:                       # 4-byte layout (PCPM_WIDE_IDS)
            np.testing.assert_array_equal(lay_gpu["ids"], ids)
            np.testing.assert_array_equal(lay_gpu["png_src"], ref.png_src)
        # compact layout = the same bins re-encoded: (v & (q-1)) | flag << 15, u & (q-1)
        # (q = 2^16 handles iterate on the 4-byte IDs; their 2-byte array keeps 15 local bits + the flag)
        want16 = ((ids & qmask & np.uint32(0x7FFF)) | ((ids >> np.uint32(31)) << np.uint32(15))).astype(np.uint16)
        np.testing.assert_array_equal(lay_gpu["ids16"], want16)
        np.testing.assert_array_equal(lay_gpu["png_src16"], (ref.png_src & qmask).astype(np.uint16))
        np.testing.assert_array_equal(lay_gpu["png_off"], ref.png_off.astype(np.uint32))
        np.testing.assert_array_equal(lay_gpu["upd_off"], ref.upd_off.astype(np.uint32))
        np.testing.assert_array_equal(lay_gpu["bin_upd_start"], ref.bin_upd_start.astype(np.uint32))
    np.testing.assert_array_equal(lay_gpu["bin_id_start"], ref.bin_id_start.astype(np.uint32))
    if g.values is not None:
        np.testing.assert_array_equal(lay_gpu["w"], ref.w)
    # decode anchors by their plain definition: #flags in ids[0 .. 128 c)
    flags = (lay_gpu["ids16"] >> 15).astype(np.int64)
    cum = np.concatenate([[0], np.cumsum(flags)])
    cb = lay_gpu["chunk_base"]
    for c in range(len(cb)):
        assert cb[c] == cum[min(128 * c, len(flags))]
    np.testing.assert_array_equal(lay_gpu["out_degree"], np.diff(g.row_ptr).astype(np.uint32))
    return ref


def g_toy():
    t = json.load(open(os.path.join(GOLDEN, "g_toy_layout.json")))
    return graphs.GraphCSR("g_toy", t["n"], t["n"], np.array(t["row_ptr"], dtype=np.int64),
                           np.array(t["col"], dtype=np.uint32))


def star_graph(n_leaves, hub=0, inward=False):
    n = n_leaves + 1
    if inward:
        rp = np.concatenate([[0, 0], np.arange(1, n_leaves + 1)]).astype(np.int64)
        col = np.zeros(n_leaves, dtype=np.uint32)
    else:
        rp = np.concatenate([[0], np.full(n, n_leaves)]).astype(np.int64)
        col = np.arange(1, n, dtype=np.uint32)
    return graphs.GraphCSR("star", n, n, rp, col)


LAYOUT_CASES = [
    ("g_toy", lambda: g_toy(), 1),
    ("c1", lambda: graphs.make_config("c1"), 8),
    ("rmat12_b4", lambda: graphs.make_graph("rmat", 7, scale=12, permute=True), 4),
    ("rmat12_b8", lambda: graphs.make_graph("rmat", 7, scale=12, permute=True), 8),
    ("rmat13_b11", lambda: graphs.make_graph("rmat", 8, scale=13, permute=False), 11),
    ("er3000_b7", lambda: graphs.make_graph("er", 5, n=3000, m_raw=50000), 7),
    ("er_ragged_b15", lambda: graphs.make_graph("er", 6, n=70001, m_raw=600000), 15),
    ("outstar_b10", lambda: star_graph(100000), 10),
    ("instar_b3", lambda: star_graph(5000, inward=True), 3),
    ("edgeless", lambda: graphs.GraphCSR("e", 100, 100, np.zeros(101, np.int64), np.zeros(0, np.uint32)), 4),
    ("self_loop", lambda: graphs.GraphCSR("s", 1, 1, np.array([0, 1], np.int64), np.array([0], np.uint32)), 1),
]


@pytest.mark.parametrize("name,mk,b", LAYOUT_CASES, ids=[c[0] for c in LAYOUT_CASES])
def test_layout_bit_exact(pcpm, name, mk, b):
    g = mk()
    h = build(pcpm, g, b)
    try:
        assert_layout_equal(g, export(pcpm, h), b)
    finally:
        pcpm.pcpm_destroy(h)


def test_layout_from_host_pointers_and_weights(pcpm):
    g = graphs.make_graph("rmat", 9, scale=11, permute=True, values=True, transpose=True)
    h = build(pcpm, g, 6, device=False)
    try:
        lay = export(pcpm, h)
        assert lay["info"].weighted == 1
        assert_layout_equal(g, lay, 6)
    finally:
        pcpm.pcpm_destroy(h)


def test_layout_uncompressed(pcpm):
    g = graphs.make_graph("rmat", 3, scale=11, permute=True)
    h = build(pcpm, g, 6, flags=pcpm.PCPM_NO_COMPRESS | pcpm.PCPM_WIDE_IDS)
    try:
        lay = export(pcpm, h)
        assert lay["info"].e_prime == g.m and lay["info"].compressed == 0
        ref = oracle.layout(g.n_src, g.n_dst, g.row_ptr, g.col, 6)
        np.testing.assert_array_equal(lay["ids"], ref.ids | np.uint32(0x80000000))
        np.testing.assert_array_equal(lay["ids16"] >> 15, np.ones(g.m, np.uint16))
        np.testing.assert_array_equal(lay["bin_id_start"], ref.bin_id_start.astype(np.uint32))
        # the uncompressed layout computes the same PageRank (every ID carries its own update)
        out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, 0.85, 10, out)
        pr_check(out.cpu().numpy(), oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, 10), "nocompress")
    finally:
        pcpm.pcpm_destroy(h)


@pytest.mark.parametrize("name,mk,b", [LAYOUT_CASES[i] for i in (1, 3, 6, 7, 9)],
                         ids=[LAYOUT_CASES[i][0] for i in (1, 3, 6, 7, 9)])
def test_layout_bit_exact_wide(pcpm, name, mk, b):
    g = mk()
    h = build(pcpm, g, b, flags=pcpm.PCPM_WIDE_IDS)
    try:
        lay = export(pcpm, h)
        assert lay["view"].wide == 1 and lay["ids"] is not None
        assert_layout_equal(g, lay, b)
    finally:
        pcpm.pcpm_destroy(h)


def test_bad_csr_rejected(pcpm):
    rp = np.array([0, 2, 3], dtype=np.int64)
    for col, code in [(np.array([1, 0, 0], np.uint32), pcpm.PCPM_EBADCSR),    # unsorted row
                      (np.array([1, 1, 0], np.uint32), pcpm.PCPM_EBADCSR),    # duplicate
                      (np.array([0, 5, 0], np.uint32), pcpm.PCPM_EBADCSR)]:   # col >= n
        with pytest.raises(pcpm.PcpmError) as e:
            pcpm.pcpm_build(pcpm.make_csr(2, 2, rp, col), 1)
        assert e.value.code == code
    rp_bad = np.array([0, 3, 2], dtype=np.int64)
    with pytest.raises(pcpm.PcpmError) as e:
        pcpm.pcpm_build(pcpm.make_csr(2, 2, rp_bad, np.array([0, 1], np.uint32)), 1)
    assert e.value.code == pcpm.PCPM_EBADCSR


@pytest.mark.parametrize("variant", [0, 3], ids=["scatter_v0", "scatter_v3_vec4"])
@pytest.mark.parametrize("name,mk,b", LAYOUT_CASES[:7], ids=[c[0] for c in LAYOUT_CASES[:7]])
def test_scatter_bit_exact(pcpm, name, mk, b, variant):
    g = mk()
    h = build(pcpm, g, b)
    try:
        pcpm.pcpm_set_option(h, "scatter_variant", variant)
        x = np.random.default_rng(1).random(g.n_src).astype(np.float32)
        xd = torch.from_numpy(x).cuda()
        pcpm.pcpm_scatter(h, xd)
        torch.cuda.synchronize()
        v = pcpm.pcpm_export_layout(h)
        info = pcpm.pcpm_get_info(h)
        got = d2h(v.upd, info.e_prime, np.float32)
        ref = oracle.scatter(oracle.layout(g.n_src, g.n_dst, g.row_ptr, g.col, b), x)
        np.testing.assert_array_equal(got.view(np.uint32), ref.view(np.uint32))
    finally:
        pcpm.pcpm_destroy(h)


def pr_check(got, ref, tag=""):
    rel = np.abs(got.astype(np.float64) - ref) / ref
    l1 = np.abs(got.astype(np.float64) - ref).sum()
    assert rel.max() <= 1e-5, f"{tag} max rel {rel.max():.3e} at {rel.argmax()}"
    assert l1 <= 1e-6, f"{tag} L1 {l1:.3e}"
    return rel.max(), l1


PR_CASES = [
    ("g_toy", lambda: g_toy(), 1, 20),
    ("c1", lambda: graphs.make_config("c1"), 8, 10),
    ("rmat14_b10", lambda: graphs.make_graph("rmat", 12, scale=14, permute=True), 10, 20),
    ("rmat15_b15", lambda: graphs.make_graph("rmat", 13, scale=15, permute=False), 15, 20),
    ("er_ragged_b15", lambda: graphs.make_graph("er", 6, n=70001, m_raw=600000), 15, 20),
    ("outstar", lambda: star_graph(20000), 12, 7),
    ("instar", lambda: star_graph(20000, inward=True), 9, 7),
    ("edgeless", lambda: graphs.GraphCSR("e", 100, 100, np.zeros(101, np.int64), np.zeros(0, np.uint32)), 4, 5),
    ("cycle", lambda: graphs.GraphCSR("c", 1000, 1000, np.arange(1001, dtype=np.int64),
                                      ((np.arange(1000) + 1) % 1000).astype(np.uint32)), 5, 20),
]


@pytest.mark.parametrize("wide", [False, True], ids=["compact", "wide"])
@pytest.mark.parametrize("name,mk,b,iters", PR_CASES, ids=[c[0] for c in PR_CASES])
def test_pagerank_parity(pcpm, name, mk, b, iters, wide):
    g = mk()
    h = build(pcpm, g, b, flags=pcpm.PCPM_BUILD_PULL | (pcpm.PCPM_WIDE_IDS if wide else 0))
    try:
        ref = oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, iters)
        out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, 0.85, iters, out)
        got = out.cpu().numpy()
        pr_check(got, ref, name)
        # bit-reproducible (fixed-point accumulation is order independent)
        out2 = torch.zeros_like(out)
        pcpm.pcpm_pagerank(h, 0.85, iters, out2)
        assert torch.equal(out, out2)
        # host output pointer
        host = np.zeros(g.n_src, dtype=np.float32)
        pcpm.pcpm_pagerank(h, 0.85, iters, host)
        np.testing.assert_array_equal(host, got)
        # the pull comparison kernel computes the same vector
        pull = torch.zeros_like(out)
        pcpm.pcpm_pull_pagerank(h, 0.85, iters, pull)
        pr_check(pull.cpu().numpy(), ref, name + "/pull")
    finally:
        pcpm.pcpm_destroy(h)


def test_pagerank_residuals_and_dangling_mass(pcpm):
    g = graphs.make_graph("rmat", 12, scale=13, permute=True)
    h = build(pcpm, g, 9)
    try:
        iters = 6
        out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, 0.85, iters, out)
        red = pcpm.pcpm_get_residuals(h)
        deg = np.diff(g.row_ptr)
        prs = [oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, t) for t in range(iters + 1)]
        for t in range(iters):
            D = prs[t][deg == 0].sum()
            assert red[2 * t] == pytest.approx(D, rel=1e-5)
            res = np.abs(prs[t + 1] - prs[t]).sum()
            assert red[2 * t + 1] == pytest.approx(res, rel=1e-3, abs=1e-7)
    finally:
        pcpm.pcpm_destroy(h)


def test_pagerank_iters_zero_and_invalid(pcpm):
    g = graphs.make_config("c1")
    h = build(pcpm, g, 8)
    try:
        out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, 0.85, 0, out)
        assert torch.all(out == 1.0 / g.n_src)
        with pytest.raises(pcpm.PcpmError):
            pcpm.pcpm_pagerank(h, 1.5, 3, out)
        with pytest.raises(pcpm.PcpmError):
            pcpm.pcpm_pull_pagerank(h, 0.85, 3, out)   # built without PCPM_BUILD_PULL
    finally:
        pcpm.pcpm_destroy(h)


def spmv_check(g, got, x, fbits):
    ref = oracle.spmv_t(g.n_src, g.n_dst, g.row_ptr, g.col, g.values, x)
    absval = None if g.values is None else np.abs(g.values)
    mag = oracle.spmv_t(g.n_src, g.n_dst, g.row_ptr, g.col, absval, np.abs(x))
    indeg = np.bincount(g.col.astype(np.int64), minlength=g.n_dst)
    # R19: each term is rounded to the 2^-F fixed-point grid (<= 2^-(F+1) each), the
    # sum is exact, and the fp32 output rounds once (<= 2^-24 |y| <= 1e-5 sum|a x|).
    tol = 1e-5 * mag + indeg * 2.0 ** (-fbits - 1) + 1e-30
    err = np.abs(got.astype(np.float64) - ref)
    assert np.all(err <= tol), f"worst {np.max(err / tol):.3f}x tol at {np.argmax(err / tol)}"


SPMV_CASES = [
    ("rmat12_w", lambda: graphs.make_graph("rmat", 5, scale=12, permute=True, values=True, transpose=True), 8),
    ("rmat15_w_b15", lambda: graphs.make_graph("rmat", 5, scale=15, permute=True, values=True, transpose=True), 15),
    ("rmat12_unweighted", lambda: graphs.make_graph("rmat", 4, scale=12, permute=True), 6),
]


@pytest.mark.parametrize("wide", [False, True], ids=["compact", "wide"])
@pytest.mark.parametrize("name,mk,b", SPMV_CASES, ids=[c[0] for c in SPMV_CASES])
def test_spmv_parity(pcpm, name, mk, b, wide):
    g = mk()
    h = build(pcpm, g, b, flags=pcpm.PCPM_WIDE_IDS if wide else 0)
    try:
        x = graphs.make_x(g.n_src, 5)
        y = torch.zeros(g.n_dst, dtype=torch.float32, device="cuda")
        pcpm.pcpm_spmv(h, torch.from_numpy(x).cuda(), y)
        fb = spmv_fbits(g.values, x)                   # from the inputs (R22), not from the library
        assert pcpm.pcpm_get_info(h).fixed_point_bits == fb
        spmv_check(g, y.cpu().numpy(), x, fb)
        yh = np.zeros(g.n_dst, dtype=np.float32)
        pcpm.pcpm_spmv(h, x, yh)                       # host pointers (fp32 order may differ: R19)
        spmv_check(g, yh, x, fb)
    finally:
        pcpm.pcpm_destroy(h)


def test_spmv_non_square(pcpm):
    rng = np.random.default_rng(3)
    ns, nd = 5000, 1300
    dens = 0.004
    rows, cols = np.nonzero(rng.random((ns, nd)) < dens)
    rp = np.zeros(ns + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    vals = rng.uniform(-1, 1, len(cols)).astype(np.float32)
    g = graphs.GraphCSR("ns", ns, nd, rp, cols.astype(np.uint32), vals)
    h = build(pcpm, g, 7)
    try:
        x = rng.uniform(-1, 1, ns).astype(np.float32)
        y = np.zeros(nd, dtype=np.float32)
        pcpm.pcpm_spmv(h, x, y)
        spmv_check(g, y, x, spmv_fbits(g.values, x))
        with pytest.raises(pcpm.PcpmError) as e:
            pcpm.pcpm_pagerank(h, 0.85, 2, np.zeros(ns, np.float32))
        assert e.value.code == pcpm.PCPM_ESTATE
    finally:
        pcpm.pcpm_destroy(h)


@pytest.mark.parametrize("opts", [{"scatter_variant": 1}, {"scatter_variant": 2}, {"scatter_variant": 3}, {"scatter_lpt": 1}, {"gather_prefetch": 0},
                                  {"cluster_gather": 0}, {"gather_variant": 2},
                                  {"gather_variant": 3, "cluster_gather": 0},
                                  {"epilogue_prefetch": 0}, {"gather_prefetch": 8, "epilogue_prefetch": 16},
                                  {"use_graph": 0}],
                         ids=lambda o: ",".join(f"{k}={v}" for k, v in o.items()))
def test_kernel_variants_keep_parity(pcpm, opts):
    """Every A/B kernel variant of DESIGN.md's design-evidence table stays oracle-exact."""
    g = graphs.make_graph("rmat", 12, scale=14, permute=True)
    h = build(pcpm, g, 10)
    try:
        for k, v in opts.items():
            pcpm.pcpm_set_option(h, k, v)
        ref = oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, 12)
        out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, 0.85, 12, out)
        pr_check(out.cpu().numpy(), ref, str(opts))
        x = graphs.make_x(g.n_src, 5)
        pcpm.pcpm_scatter(h, torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        v = pcpm.pcpm_export_layout(h)
        info = pcpm.pcpm_get_info(h)
        got = d2h(v.upd, info.e_prime, np.float32)
        want = oracle.scatter(oracle.layout(g.n_src, g.n_dst, g.row_ptr, g.col, 10), x)
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    finally:
        pcpm.pcpm_destroy(h)


PA_CASES = [
    ("rmat18_b11", lambda: graphs.make_graph("rmat", 21, scale=18, permute=True), 11),
    ("rmat20_b15", lambda: graphs.make_graph("rmat", 22, scale=20, permute=True), 15),
    ("rmat19_bfs_b13", lambda: graphs.make_graph("rmat", 23, scale=19, permute=False), 13),
    ("er_ragged_b9", lambda: graphs.make_graph("er", 6, n=70001, m_raw=600000), 9),
]


@pytest.mark.parametrize("name,mk,b", PA_CASES, ids=[c[0] for c in PA_CASES])
def test_producer_apply_bit_identical(pcpm, name, mk, b):
    """gather_variant 3 (the apply in the producer warps from tensor memory) gives the
    oracle's PageRank within the BASELINE bounds and the same bits as the in-line
    epilogue (both sum the same integers), including split bins, a ragged last partition
    and the residual / dangling reductions."""
    g = mk()
    h = build(pcpm, g, b)
    try:
        pcpm.pcpm_set_option(h, "cluster_gather", 0)
        iters = 9
        outs, res = [], []
        for var in (1, 3):
            pcpm.pcpm_set_option(h, "gather_variant", var)
            out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
            pcpm.pcpm_pagerank(h, 0.85, iters, out)
            torch.cuda.synchronize()
            outs.append(out.cpu().numpy())
            res.append(np.asarray(pcpm.pcpm_get_residuals(h, iters)))
        np.testing.assert_array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
        np.testing.assert_array_equal(res[0], res[1])
        ref = oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, iters)
        pr_check(outs[1], ref, name)
    finally:
        pcpm.pcpm_destroy(h)


CHUNK_CASES = [
    ("c1", lambda: graphs.make_config("c1"), 8, False, 0),
    ("rmat13_b6_host", lambda: graphs.make_graph("rmat", 8, scale=13, permute=True), 6, True, 0),
    ("rmat12_b4_weights", lambda: graphs.make_graph("rmat", 9, scale=12, permute=True, values=True,
                                                    transpose=True), 4, True, 0),
    ("er_ragged_b9_wide", lambda: graphs.make_graph("er", 6, n=70001, m_raw=600000), 9, False, 8),
    ("outstar_b5", lambda: star_graph(20000), 5, True, 0),
    ("rmat11_b3_nocompress", lambda: graphs.make_graph("rmat", 3, scale=11, permute=True), 3, False, 1),
]


@pytest.mark.parametrize("name,mk,b,host,flags", CHUNK_CASES, ids=[c[0] for c in CHUNK_CASES])
@pytest.mark.parametrize("mode", ["count", "count_seg1", "count_seg200", "count_onelevel", "warp", "warp_seg200",
                                  "sort_1", "sort_777", "legacy", "default"])
def test_layout_chunked_build(pcpm, monkeypatch, name, mk, b, host, flags, mode):
    """Every construction gives the oracle's layout, for host or device inputs, weights,
    wide IDs and uncompressed bins: the counting build (default; segments of one
    32-row batch with PCPM_BUILD_SEG_EDGES=1, ~200 edges, or the default plan), the
    chunked sort for any chunk size (PCPM_BUILD=sort), and the legacy path.  The counting
    build places in two levels (segment buckets, then bins) when k_dst > 64 and in one level
    with PCPM_BUILD_ONE_LEVEL=1; "default" leaves the choice to pcpm_build (host inputs:
    the chunked sort)."""
    if mode.startswith("count") or mode.startswith("warp"):
        monkeypatch.setenv("PCPM_BUILD", "count")    # also for host inputs
    if mode == "count_onelevel":
        monkeypatch.setenv("PCPM_BUILD_ONE_LEVEL", "1")
    if mode == "legacy":
        monkeypatch.setenv("PCPM_BUILD_LEGACY", "1")
    elif mode.startswith("sort_"):
        monkeypatch.setenv("PCPM_BUILD", "sort")
        monkeypatch.setenv("PCPM_BUILD_CHUNK_EDGES", mode[5:])
    elif mode.startswith("count_seg"):
        monkeypatch.setenv("PCPM_BUILD_SEG_EDGES", mode[9:])
    elif mode.startswith("warp"):                    # the warp-per-segment form of the counting build
        monkeypatch.setenv("PCPM_BUILD_COUNT_MODE", "warp")
        if mode == "warp_seg200":
            monkeypatch.setenv("PCPM_BUILD_SEG_EDGES", "200")
    g = mk()
    h = build(pcpm, g, b, device=not host, flags=flags)
    try:
        lay = export(pcpm, h)
        if flags & 1:                          # PCPM_NO_COMPRESS: every ID flagged
            ref = oracle.layout(g.n_src, g.n_dst, g.row_ptr, g.col, b)
            assert lay["info"].e_prime == g.m
            np.testing.assert_array_equal(lay["ids16"] >> 15, np.ones(g.m, np.uint16))
            np.testing.assert_array_equal(lay["ids16"] & np.uint16(0x7FFF),
                                          (ref.ids & np.uint32((1 << b) - 1)).astype(np.uint16))
            np.testing.assert_array_equal(lay["bin_id_start"], ref.bin_id_start.astype(np.uint32))
        else:
            assert_layout_equal(g, lay, b)
    finally:
        pcpm.pcpm_destroy(h)


def weighted(g, seed, zero_frac=0.1):
    """g with non-negative fp32 edge weights (some exactly zero) for weighted PageRank."""
    rng = np.random.default_rng(seed)
    w = rng.uniform(0.0, 1.0, g.m).astype(np.float32)
    w[rng.random(g.m) < zero_frac] = 0.0
    return graphs.GraphCSR(g.name + "_w", g.n_src, g.n_dst, g.row_ptr, g.col, w)


WPR_CASES = [
    ("rmat12_b8", lambda: weighted(graphs.make_graph("rmat", 12, scale=12, permute=True), 1), 8, True),
    ("rmat14_b10_host", lambda: weighted(graphs.make_graph("rmat", 13, scale=14, permute=True), 2), 10, False),
    ("rmat15_b15_split", lambda: weighted(graphs.make_graph("rmat", 13, scale=15, permute=False), 3), 15, True),
    ("er_ragged_b9", lambda: weighted(graphs.make_graph("er", 6, n=70001, m_raw=600000), 4, 0.3), 9, True),
]


@pytest.mark.parametrize("name,mk,b,device", WPR_CASES, ids=[c[0] for c in WPR_CASES])
def test_weighted_pagerank_parity(pcpm, name, mk, b, device):
    """Weighted PageRank (R24): the gather applies w(u,v) to the source value,
    the apply normalises by W(u); oracle bounds as for Eq. 1, bit-reproducible."""
    g = mk()
    h = build(pcpm, g, b, device=device)
    try:
        pcpm.pcpm_set_option(h, "weighted_pagerank", 1)
        ref = oracle.pagerank_weighted(g.n_src, g.row_ptr, g.col, g.values, 0.85, 15)
        out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, 0.85, 15, out)
        pr_check(out.cpu().numpy(), ref, name)
        out2 = torch.zeros_like(out)
        pcpm.pcpm_pagerank(h, 0.85, 15, out2)
        assert torch.equal(out, out2)
        pcpm.pcpm_set_option(h, "weighted_pagerank", 0)     # back to Eq. 1 on the structure
        pcpm.pcpm_pagerank(h, 0.85, 15, out)
        pr_check(out.cpu().numpy(), oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, 15), name + "/unweighted")
    finally:
        pcpm.pcpm_destroy(h)


def test_weighted_pagerank_rejected_without_usable_weights(pcpm):
    g = graphs.make_graph("rmat", 12, scale=10, permute=True)
    h = build(pcpm, g, 6)
    try:
        with pytest.raises(pcpm.PcpmError) as e:
            pcpm.pcpm_set_option(h, "weighted_pagerank", 1)        # no values
        assert e.value.code == pcpm.PCPM_ESTATE
    finally:
        pcpm.pcpm_destroy(h)
    gs = graphs.make_graph("rmat", 5, scale=10, permute=True, values=True)   # values in [-1, 1)
    h = build(pcpm, gs, 6)
    try:
        with pytest.raises(pcpm.PcpmError) as e:
            pcpm.pcpm_set_option(h, "weighted_pagerank", 1)
        assert e.value.code == pcpm.PCPM_EINVAL
    finally:
        pcpm.pcpm_destroy(h)


@pytest.mark.parametrize("tol", [1e-4, 1e-6])
def test_pagerank_to_tolerance(pcpm, tol):
    """pcpm_pagerank_tol stops at the first t whose L1 residual sum|PR_t - PR_{t-1}| <= tol
    and returns exactly pcpm_pagerank's PR_t (the same kernels)."""
    g = graphs.make_graph("rmat", 12, scale=14, permute=True)
    h = build(pcpm, g, 10)
    try:
        out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        t = pcpm.pcpm_pagerank_tol(h, 0.85, tol, 200, out)
        assert 1 <= t < 200
        prs = [oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, k) for k in (t - 1, t)]
        pr_check(out.cpu().numpy(), prs[1], "tol")
        res = np.abs(prs[1] - prs[0]).sum()
        assert res <= tol * 1.01 + 1e-7                  # fp32 vs fp64 residual
        if t >= 2:
            prev = np.abs(prs[0] - oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, t - 2)).sum()
            assert prev >= tol * 0.99 - 1e-7               # it did not stop early
        ref = torch.zeros_like(out)
        pcpm.pcpm_pagerank(h, 0.85, t, ref)
        assert torch.equal(out, ref)
        host = np.zeros(g.n_src, np.float32)
        assert pcpm.pcpm_pagerank_tol(h, 0.85, 0.0, 7, host) == 7      # tol 0: runs max_iters
        pcpm.pcpm_pagerank(h, 0.85, 7, ref)
        np.testing.assert_array_equal(host, ref.cpu().numpy())
        with pytest.raises(pcpm.PcpmError):
            pcpm.pcpm_pagerank_tol(h, 0.85, -1.0, 5, out)
    finally:
        pcpm.pcpm_destroy(h)


def test_pipelined_jobs_match_single_build(pcpm):
    """bench.py's e2e schedule: CSR uploaded on a copy stream while the previous job
    iterates, built from the device copy on a compute stream (nnz passed from the host),
    result downloaded on a third stream -- every job's PR is bit-identical to a plain
    build + pcpm_pagerank; pcpm_pool_reserve leaves the pool usable."""
    g = graphs.make_graph("rmat", 21, scale=13, permute=True)
    assert pcpm.pcpm_pool_reserve(64 << 20) == pcpm.PCPM_OK
    h = build(pcpm, g, 10)
    try:
        ref = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, 0.85, 12, ref)
        ref = ref.cpu()
    finally:
        pcpm.pcpm_destroy(h)
    rp = torch.from_numpy(np.ascontiguousarray(g.row_ptr)).pin_memory()
    col = torch.from_numpy(np.ascontiguousarray(g.col).view(np.int32)).pin_memory()
    comp, h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    stage = [(torch.empty_like(rp, device="cuda"), torch.empty_like(col, device="cuda")) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    dev = [torch.zeros(g.n_src, device="cuda") for _ in range(2)]
    outs = []
    prev = None
    for k in range(3):
        h2d.wait_stream(comp)
        with torch.cuda.stream(h2d):
            stage[k & 1][0].copy_(rp, non_blocking=True)
            stage[k & 1][1].copy_(col, non_blocking=True)
            ready[k & 1].record(h2d)
        comp.wait_event(ready[k & 1])
        if prev is not None:
            pcpm.pcpm_destroy(prev)
        csr = pcpm.make_csr(g.n_src, g.n_dst, stage[k & 1][0], stage[k & 1][1], None, nnz=int(rp[-1]))
        prev = pcpm.pcpm_build_ex(csr, 10, 0, comp)
        with torch.cuda.stream(comp):
            pcpm.pcpm_pagerank(prev, 0.85, 12, dev[k & 1])
        d2h.wait_stream(comp)
        host = torch.empty(g.n_src, pin_memory=True)
        with torch.cuda.stream(d2h):
            host.copy_(dev[k & 1], non_blocking=True)
        outs.append(host)
    pcpm.pcpm_destroy(prev)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)


@pytest.mark.parametrize("scale,b", [(16, 8), (17, 9)])
def test_compact_slots_match(pcpm, scale, b):
    """PCPM_COMPACT_SLOTS (accumulator slots = rank among the partition's vertices with
    in-edges, 6-stage gather ring): PageRank and SpMV bit-identical to the default layout
    and within the oracle bounds; the remapped IDs equal the oracle's local IDs mapped
    through the per-partition ranks computed here from the oracle layout."""
    g = graphs.make_graph("rmat", 31, scale=scale, permute=True)
    h0 = build(pcpm, g, b)
    h1 = build(pcpm, g, b, pcpm.PCPM_COMPACT_SLOTS)
    try:
        assert pcpm.pcpm_get_info(h1).compact_slots == 1, "slots not applied"
        outs = []
        for h in (h0, h1):
            o = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
            pcpm.pcpm_pagerank(h, 0.85, 15, o)
            outs.append(o.cpu())
        assert torch.equal(outs[0], outs[1])
        pr_check(outs[1].numpy(), oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, 15), "slots")
        x = torch.from_numpy(graphs.make_x(g.n_src, 31)).cuda()
        ys = []
        for h in (h0, h1):
            y = torch.zeros(g.n_dst, dtype=torch.float32, device="cuda")
            pcpm.pcpm_spmv(h, x, y)
            ys.append(y.cpu())
        assert torch.equal(ys[0], ys[1])
        # IDs: slot = rank of the local ID among vertices with in-edges in its partition
        ref = oracle.layout(g.n_src, g.n_dst, g.row_ptr, g.col, b)
        q = 1 << b
        has_in = np.zeros(((g.n_dst + q - 1) // q) * q, dtype=bool)
        has_in[np.asarray(g.col, dtype=np.int64)] = True
        rank = (np.cumsum(has_in.reshape(-1, q), axis=1) - 1).reshape(-1)
        ids_o = np.asarray(ref.ids, dtype=np.uint32)
        v = (ids_o & np.uint32(0x7FFFFFFF)).astype(np.int64)
        want = (rank[v].astype(np.uint32) | ((ids_o >> np.uint32(31)) << np.uint32(15))).astype(np.uint16)
        np.testing.assert_array_equal(export(pcpm, h1)["ids16"], want)
    finally:
        pcpm.pcpm_destroy(h0)
        pcpm.pcpm_destroy(h1)


def test_compact_slots_ragged_partition(pcpm):
    """Slots with a short last partition (n not a multiple of q or of 4): the scalar apply
    path; PageRank identical to the default layout."""
    g = graphs.make_graph("er", 33, n=3 * 4096 * 8 + 3, m_raw=400000)
    h0 = build(pcpm, g, 8)
    h1 = build(pcpm, g, 8, pcpm.PCPM_COMPACT_SLOTS)
    try:
        outs = []
        for h in (h0, h1):
            o = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
            pcpm.pcpm_pagerank(h, 0.85, 9, o)
            outs.append(o.cpu())
        assert torch.equal(outs[0], outs[1])
    finally:
        pcpm.pcpm_destroy(h0)
        pcpm.pcpm_destroy(h1)


def test_job_runtime_matches_oracle_and_single_calls(pcpm):
    """pcpm_runtime / pcpm_job_*: jobs from host memory (H2D, build, iterations, D2H), run
    back to back by the native worker with uploads overlapping compute, give the same PR
    as one pcpm_build + pcpm_pagerank per graph (bit for bit) and match the oracle."""
    ga = graphs.make_graph("rmat", 12, scale=13, permute=True)
    gb = graphs.make_graph("er", 9, n=30001, m_raw=300000)
    jobs = [(ga, 9, 10), (gb, 11, 7), (ga, 9, 10), (gb, 6, 3)]
    rt = pcpm.pcpm_runtime_create()
    try:
        keep, ids, outs = [], [], []
        for g, b, it in jobs:
            rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
            col = np.ascontiguousarray(g.col, dtype=np.uint32)
            out = np.zeros(g.n_src, dtype=np.float32)
            keep.append((rp, col))
            outs.append(out)
            ids.append(pcpm.pcpm_job_submit(rt, pcpm.make_csr(g.n_src, g.n_dst, rp, col), b, 0, 0.85, it, out))
        for i in reversed(ids):                  # any wait order
            pcpm.pcpm_job_wait(rt, i)
        with pytest.raises(pcpm.PcpmError):
            pcpm.pcpm_job_wait(rt, ids[0])       # already waited for
        for (g, b, it), out in zip(jobs, outs):
            h = build(pcpm, g, b)
            try:
                single = np.zeros(g.n_src, dtype=np.float32)
                pcpm.pcpm_pagerank(h, 0.85, it, single)
            finally:
                pcpm.pcpm_destroy(h)
            np.testing.assert_array_equal(out.view(np.uint32), single.view(np.uint32))
            pr_check(out, oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, it), "job")
        # a failing job reports its error and the runtime keeps working
        bad_rp = np.array([0, 2, 3], dtype=np.int64)
        bad_col = np.array([1, 0, 0], dtype=np.uint32)        # unsorted row: PCPM_EBADCSR
        out = np.zeros(2, dtype=np.float32)
        j = pcpm.pcpm_job_submit(rt, pcpm.make_csr(2, 2, bad_rp, bad_col), 1, 0, 0.85, 2, out)
        with pytest.raises(pcpm.PcpmError) as e:
            pcpm.pcpm_job_wait(rt, j)
        assert e.value.code == pcpm.PCPM_EBADCSR
        g, b, it = jobs[1]
        out = np.zeros(g.n_src, dtype=np.float32)
        j = pcpm.pcpm_job_submit(rt, pcpm.make_csr(g.n_src, g.n_dst, keep[1][0], keep[1][1]), b, 0, 0.85, it, out)
        pcpm.pcpm_job_wait(rt, j)
        np.testing.assert_array_equal(out, outs[1])
    finally:
        pcpm.pcpm_runtime_destroy(rt)


FUSE_CASES = [
    ("rmat14_b6", lambda: graphs.make_graph("rmat", 12, scale=14, permute=True), 6, False),
    ("rmat15_unpermuted_b7", lambda: graphs.make_graph("rmat", 13, scale=15, permute=False), 7, False),  # hub bins: split
    ("er_ragged_b9", lambda: graphs.make_graph("er", 6, n=70001, m_raw=600000), 9, False),
    ("rmat14_weighted_b6", lambda: weighted(graphs.make_graph("rmat", 12, scale=14, permute=True), 4), 6, True),
]


@pytest.mark.parametrize("name,mk,b,wpr", FUSE_CASES, ids=[c[0] for c in FUSE_CASES])
def test_fused_iteration_matches_unfused_and_oracle(pcpm, name, mk, b, wpr):
    """The fused iteration (each gather kernel also scatters the next iteration's updates from the
    SPR values it keeps on chip; split partitions scattered after k_apply_split) computes the
    same PageRank, bit for bit, as separate scatter and gather kernels, and matches the oracle."""
    g = mk()
    h = build(pcpm, g, b)
    try:
        if wpr:
            pcpm.pcpm_set_option(h, "weighted_pagerank", 1)
        outs = {}
        for fuse in (1, 0):                       # the fused iteration is opt-in (measured slower)
            pcpm.pcpm_set_option(h, "fuse_scatter", fuse)
            out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
            pcpm.pcpm_pagerank(h, 0.85, 9, out)
            torch.cuda.synchronize()
            assert pcpm.pcpm_get_info(h).fused_iterations == fuse
            outs[fuse] = (out.cpu().numpy(), pcpm.pcpm_get_residuals(h))
        np.testing.assert_array_equal(outs[1][0].view(np.uint32), outs[0][0].view(np.uint32))
        np.testing.assert_array_equal(outs[1][1], outs[0][1])
        ref = (oracle.pagerank_weighted(g.n_src, g.row_ptr, g.col, g.values, 0.85, 9) if wpr
               else oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, 9))
        pr_check(outs[1][0], ref, name)
    finally:
        pcpm.pcpm_destroy(h)


BVGAS_CASES = [
    ("c1", lambda: graphs.make_config("c1"), 8),
    ("rmat12_b4", lambda: graphs.make_graph("rmat", 7, scale=12, permute=True), 4),
    ("rmat13_b6", lambda: graphs.make_graph("rmat", 8, scale=13, permute=True), 6),
    ("er_ragged_b15", lambda: graphs.make_graph("er", 6, n=70001, m_raw=600000), 15),
    ("outstar_b10", lambda: star_graph(100000), 10),
    ("instar_b3", lambda: star_graph(5000, inward=True), 3),
]


@pytest.mark.parametrize("name,mk,b", BVGAS_CASES, ids=[c[0] for c in BVGAS_CASES])
def test_bvgas_engine(pcpm, name, mk, b):
    """The BVGAS comparison engine (Alg. 3): its vertex-centric scatter fills the
    uncompressed bins -- every edge (u, v) one update, bins in (v >> b, u, v) order, i.e.
    upd[x] = x[u] for the x-th edge of that order (a sort-based construction written here,
    not the kernels' counting placement) -- and its PageRank matches the oracle and is
    bit-identical to PCPM's on the same uncompressed layout."""
    g = mk()
    h = build(pcpm, g, b, flags=pcpm.PCPM_BVGAS)
    hp = build(pcpm, g, b, flags=pcpm.PCPM_NO_COMPRESS)
    try:
        info = pcpm.pcpm_get_info(h)
        assert info.bvgas == 1 and info.compressed == 0 and info.e_prime == g.m
        x = np.random.default_rng(3).random(g.n_src).astype(np.float32)
        pcpm.pcpm_scatter(h, torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        got = d2h(pcpm.pcpm_export_layout(h).upd, g.m, np.float32)
        src = np.repeat(np.arange(g.n_src, dtype=np.int64), np.diff(g.row_ptr))
        dst = g.col.astype(np.int64)
        order = np.lexsort((dst, src, dst >> b))         # bin, then u, then v
        np.testing.assert_array_equal(got.view(np.uint32), x[src[order]].view(np.uint32))
        ref = oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, 12)
        out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, 0.85, 12, out)
        outp = torch.zeros_like(out)
        pcpm.pcpm_pagerank(hp, 0.85, 12, outp)
        got_pr = out.cpu().numpy()
        pr_check(got_pr, ref, f"bvgas {name}")
        np.testing.assert_array_equal(got_pr.view(np.uint32), outp.cpu().numpy().view(np.uint32))
    finally:
        pcpm.pcpm_destroy(h)
        pcpm.pcpm_destroy(hp)


def test_bvgas_rejects(pcpm):
    g = graphs.make_graph("rmat", 9, scale=10, permute=True, values=True, transpose=True)
    with pytest.raises(pcpm.PcpmError) as e:
        build(pcpm, g, 6, flags=pcpm.PCPM_BVGAS)                 # weighted
    assert e.value.code == pcpm.PCPM_EINVAL
    gr = graphs.make_graph("er", 4, n=3000, m_raw=20000)
    rp, col = gr.row_ptr, gr.col
    with pytest.raises(pcpm.PcpmError) as e:                      # non-square
        pcpm.pcpm_build_ex(pcpm.make_csr(gr.n_src, gr.n_src + 100, rp, col), 6, pcpm.PCPM_BVGAS, None)
    assert e.value.code == pcpm.PCPM_EINVAL


# ---- q = 2^16 ("pair" handles): 4-byte IDs, two half-partition gather items per
# bin, source values read through L1/L2 in the scatter.  Layout bit-exact against the oracle at
# b = 16, PageRank / SpMV within the BASELINE bounds and -- the fixed-point sums being exact and
# order-free -- bit-identical to the b = 15 handle's results.
PAIR_CASES = [
    ("er_ragged_70001", lambda: graphs.make_graph("er", 6, n=70001, m_raw=600000)),          # k = 2, no upper half in the last
    ("er_98309", lambda: graphs.make_graph("er", 9, n=98309, m_raw=700000)),                 # upper half of 5 vertices
    ("rmat17", lambda: graphs.make_graph("rmat", 21, scale=17, permute=True)),               # k = 2 full partitions
    ("rmat18_bfs_like", lambda: graphs.make_graph("rmat", 22, scale=18, permute=False)),     # k = 4, skewed bins
    ("small_1000", lambda: graphs.make_graph("er", 3, n=1000, m_raw=8000)),                  # one partial partition
    ("instar", lambda: star_graph(150000, inward=True)),
]


@pytest.mark.parametrize("name,mk", PAIR_CASES, ids=[c[0] for c in PAIR_CASES])
def test_pair_q16_layout_and_pagerank(pcpm, name, mk):
    g = mk()
    h = build(pcpm, g, 16)
    h15 = build(pcpm, g, 15)
    try:
        lay = export(pcpm, h)
        assert lay["view"].wide == 1 and lay["ids"] is not None and lay["info"].partition_bits == 16
        assert_layout_equal(g, lay, 16)
        x = np.random.default_rng(2).random(g.n_src).astype(np.float32)
        pcpm.pcpm_scatter(h, torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        got = d2h(lay["view"].upd, lay["info"].e_prime, np.float32)
        ref_u = oracle.scatter(oracle.layout(g.n_src, g.n_dst, g.row_ptr, g.col, 16), x)
        np.testing.assert_array_equal(got.view(np.uint32), ref_u.view(np.uint32))
        ref = oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, 12)
        out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, 0.85, 12, out)
        pr_check(out.cpu().numpy(), ref, name)
        out15 = torch.zeros_like(out)
        pcpm.pcpm_pagerank(h15, 0.85, 12, out15)
        assert torch.equal(out, out15)
        # kernel options that do not apply to pair handles are ignored, not mis-run
        for k, v in (("gather_variant", 2), ("scatter_variant", 3), ("scatter_variant", 1)):
            pcpm.pcpm_set_option(h, k, v)
        out2 = torch.zeros_like(out)
        pcpm.pcpm_pagerank(h, 0.85, 12, out2)
        assert torch.equal(out, out2)
    finally:
        pcpm.pcpm_destroy(h)
        pcpm.pcpm_destroy(h15)


@pytest.mark.parametrize("name,mk", [
    ("rmat17_w", lambda: graphs.make_graph("rmat", 23, scale=17, permute=True, values=True, transpose=True)),
    ("nonsquare", lambda: graphs.column_prefix(graphs.make_graph("er", 24, n=150001, m_raw=1500000, values=True), 70003)),
], ids=["rmat17_w", "nonsquare"])
def test_pair_q16_spmv(pcpm, name, mk):
    g = mk()
    h = build(pcpm, g, 16)
    try:
        assert_layout_equal(g, export(pcpm, h), 16)
        x = graphs.make_x(g.n_src, 4)
        y = torch.zeros(g.n_dst, dtype=torch.float32, device="cuda")
        pcpm.pcpm_spmv(h, torch.from_numpy(x).cuda(), y)
        spmv_check(g, y.cpu().numpy(), x, spmv_fbits(g.values, x))
    finally:
        pcpm.pcpm_destroy(h)


def test_pair_q16_rejections(pcpm):
    g = graphs.make_graph("er", 3, n=1000, m_raw=8000)
    rp, col, _ = to_device(g)
    csr = pcpm.make_csr(g.n_src, g.n_dst, rp, col)
    for call in (lambda: pcpm.pcpm_build(csr, 17),
                 lambda: pcpm.pcpm_build_shard(csr, 16, 0, 1000, 0, None),
                 lambda: pcpm.pcpm_build_ex(csr, 16, pcpm.PCPM_BVGAS, None)):
        with pytest.raises(pcpm.PcpmError) as e:
            call()
        assert e.value.code == pcpm.PCPM_EINVAL


def test_pair_q16_variants(pcpm):
    """q = 2^16 with the other layouts and drivers: uncompressed bins, host CSR pointers,
    weighted PageRank (R24), the tolerance driver and the pipelined job runtime."""
    g = graphs.make_graph("er", 6, n=70001, m_raw=600000)
    ref = oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, 10)
    for flags, device in ((pcpm.PCPM_NO_COMPRESS, True), (0, False), (pcpm.PCPM_BUILD_PULL, True)):
        h = build(pcpm, g, 16, flags=flags, device=device)
        try:
            out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
            pcpm.pcpm_pagerank(h, 0.85, 10, out)
            pr_check(out.cpu().numpy(), ref, f"flags={flags}")
            if flags & pcpm.PCPM_BUILD_PULL:
                pull = torch.zeros_like(out)
                pcpm.pcpm_pull_pagerank(h, 0.85, 10, pull)
                pr_check(pull.cpu().numpy(), ref, "pull")
                it = pcpm.pcpm_pagerank_tol(h, 0.85, 1e-7, 100, out)
                assert 1 <= it < 100
                pr_check(out.cpu().numpy(), oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, it), "tol")
        finally:
            pcpm.pcpm_destroy(h)
    gw = weighted(graphs.make_graph("er", 6, n=70001, m_raw=600000), 4, 0.3)
    h = build(pcpm, gw, 16)
    try:
        pcpm.pcpm_set_option(h, "weighted_pagerank", 1)
        out = torch.zeros(gw.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, 0.85, 15, out)
        pr_check(out.cpu().numpy(), oracle.pagerank_weighted(gw.n_src, gw.row_ptr, gw.col, gw.values, 0.85, 15), "wpr16")
    finally:
        pcpm.pcpm_destroy(h)
