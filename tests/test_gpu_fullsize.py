"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Each config is built exactly as bench.py builds it (same generator, same
partition bits, default compact layout, the CUDA-graph PageRank of
pcpm_pagerank / the pcpm_spmv call), then the whole output vector is compared
with the fp64 oracle (oracle/, OpenMP pull form for PageRank), element by
element:
  * PageRank: max relative error <= 1e-5 and L1 <= 1e-6 (BASELINE north_star);
  * SpMV: |y - y_o| <= 1e-5 sum|a x| + indeg 2^-(F+1) per row (R22).
Plus properties that hold at any size: sum(PR) = 1 (R1), the per-iteration
dangling mass D_t and the contraction of the L1 residual (||PR_{t+1}-PR_t||
<= d ||PR_t - PR_{t-1}||).

These take minutes (c4: 1.06 B edges, the oracle needs ~1 s per iteration on
16 host cores), so they are also marked ``slow``.
"""
import numpy as np
import pytest

import oracle
from inputs import graphs

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def pcpm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1709_07122_b200 import pcpm as p
    return p


@pytest.mark.parametrize("key", ["c2", "c3", "c4", "c4bfs"])
def test_fullsize_pagerank(pcpm, key):
    cfg = graphs.CONFIGS[key]
    iters, b, d = cfg["iters"], cfg["bits"], 0.85
    g = graphs.make_config(key, backend="torch", device="cuda")
    h = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, g.row_ptr, g.col, None), b, 0,
                           torch.cuda.current_stream())
    try:
        info = pcpm.pcpm_get_info(h)
        out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
        pcpm.pcpm_pagerank(h, d, iters, out)
        torch.cuda.synchronize()
        red = pcpm.pcpm_get_residuals(h)
        got = out.cpu().numpy()
        # bit-reproducible at full size too (fixed-point accumulation)
        out2 = torch.zeros_like(out)
        pcpm.pcpm_pagerank(h, d, iters, out2)
        assert torch.equal(out, out2)
    finally:
        pcpm.pcpm_destroy(h)
    gn = g.to_numpy()
    del g
    torch.cuda.empty_cache()
    n = gn.n_src
    in_ptr, in_src = oracle.transpose(n, gn.row_ptr, gn.col)
    ref = oracle.pagerank_pull(n, gn.row_ptr, in_ptr, in_src, d, iters)
    rel = np.abs(got.astype(np.float64) - ref) / ref
    l1 = np.abs(got.astype(np.float64) - ref).sum()
    print(f"{key}: n={n} m={info.nnz} E'={info.e_prime} max_rel={rel.max():.3e} L1={l1:.3e}")
    assert rel.max() <= 1e-5, f"{key} max rel {rel.max():.3e} at {rel.argmax()}"
    assert l1 <= 1e-6, f"{key} L1 {l1:.3e}"
    # invariants
    assert abs(got.astype(np.float64).sum() - 1.0) <= 1e-5
    deg = np.diff(gn.row_ptr)
    assert red[2 * (iters - 1)] == pytest.approx(
        oracle.pagerank_pull(n, gn.row_ptr, in_ptr, in_src, d, iters - 1)[deg == 0].sum(), rel=1e-5)
    # contraction, down to the floor set by storing PR in fp32 between iterations
    # (each stored value rounds by <= 2^-24 relative, so sum |rounding| <= 2^-24)
    res = red[1::2][:iters]
    assert np.all(res[1:] <= d * res[:-1] * (1 + 1e-3) + 2.0 ** -22), res


def test_fullsize_spmv(pcpm):
    key = "c5"
    cfg = graphs.CONFIGS[key]
    g = graphs.make_config(key, backend="torch", device="cuda")
    h = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, g.row_ptr, g.col, g.values), cfg["bits"], 0,
                           torch.cuda.current_stream())
    try:
        x = graphs.make_x(g.n_src, cfg["seed"], backend="torch", device="cuda")
        y = torch.zeros(g.n_dst, dtype=torch.float32, device="cuda")
        for _ in range(3):                       # repeated multiplies (bench steps several)
            pcpm.pcpm_spmv(h, x, y)
        torch.cuda.synchronize()
        fb = pcpm.pcpm_get_info(h).fixed_point_bits
        got = y.cpu().numpy()
        xh = x.cpu().numpy()
    finally:
        pcpm.pcpm_destroy(h)
    gn = g.to_numpy()
    del g
    torch.cuda.empty_cache()
    ref = oracle.spmv_t(gn.n_src, gn.n_dst, gn.row_ptr, gn.col, gn.values, xh)
    mag = oracle.spmv_t(gn.n_src, gn.n_dst, gn.row_ptr, gn.col, np.abs(gn.values), np.abs(xh))
    indeg = np.bincount(gn.col.astype(np.int64), minlength=gn.n_dst)
    tol = 1e-5 * mag + indeg * 2.0 ** (-fb - 1) + 1e-30
    err = np.abs(got.astype(np.float64) - ref)
    print(f"{key}: nnz={gn.m} F={fb} max_abs_err={err.max():.3e} worst err/tol={np.max(err / tol):.3e}")
    assert np.all(err <= tol), f"worst {np.max(err / tol):.3f}x tol at {np.argmax(err / tol)}"


@pytest.mark.parametrize("key", ["c4", "c5"])
def test_fullsize_host_build_equals_device_build(pcpm, key):
    """The e2e path (host CSR in pinned memory: chunks copied on a second stream while
    earlier chunks sort) builds the same layout, bit for bit, as the device-input
    build, and the same PageRank / SpMV output, at full size."""
    from tests.gpu_util import d2h
    cfg = graphs.CONFIGS[key]
    g = graphs.make_config(key, backend="torch", device="cuda")
    pin = lambda t: t.cpu().pin_memory() if t is not None else None     # noqa: E731
    rp_h, col_h, val_h = pin(g.row_ptr), pin(g.col), pin(g.values)
    hd = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, g.row_ptr, g.col, g.values), cfg["bits"], 0, None)
    hh = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, rp_h, col_h, val_h), cfg["bits"], 0, None)
    try:
        ia, ib = pcpm.pcpm_get_info(hd), pcpm.pcpm_get_info(hh)
        assert (ia.nnz, ia.e_prime, ia.k_src, ia.k_dst, ia.n_dangling) == (ib.nnz, ib.e_prime, ib.k_src, ib.k_dst,
                                                                           ib.n_dangling)
        va, vb = pcpm.pcpm_export_layout(hd), pcpm.pcpm_export_layout(hh)
        m, ep, ks, kd = ia.nnz, ia.e_prime, ia.k_src, ia.k_dst
        for name, count, dt in [("ids16", m, np.uint16), ("png_src16", ep, np.uint16),
                                ("png_off", ks * (kd + 1), np.uint32), ("upd_off", ks * kd, np.uint32),
                                ("bin_id_start", kd + 1, np.uint32), ("bin_upd_start", kd + 1, np.uint32),
                                ("chunk_base", m // 128 + 1, np.uint32), ("out_degree", ia.n_src, np.uint32)] + \
                               ([("w", m, np.float32)] if g.values is not None else []):
            a, b = d2h(getattr(va, name), count, dt), d2h(getattr(vb, name), count, dt)
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), name
        if g.values is None:
            oa = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
            ob = torch.zeros_like(oa)
            pcpm.pcpm_pagerank(hd, 0.85, 3, oa)
            pcpm.pcpm_pagerank(hh, 0.85, 3, ob)
        else:
            x = graphs.make_x(g.n_src, cfg["seed"], backend="torch", device="cuda")
            oa = torch.zeros(g.n_dst, dtype=torch.float32, device="cuda")
            ob = torch.zeros_like(oa)
            pcpm.pcpm_spmv(hd, x, oa)
            pcpm.pcpm_spmv(hh, x, ob)
        torch.cuda.synchronize()
        assert torch.equal(oa, ob)
    finally:
        pcpm.pcpm_destroy(hd)
        pcpm.pcpm_destroy(hh)
