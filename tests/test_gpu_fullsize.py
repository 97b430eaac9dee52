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
from tests.gpu_util import spmv_fbits

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
        got = y.cpu().numpy()
        xh = x.cpu().numpy()
        fb = spmv_fbits(g.values.cpu().numpy(), xh)     # from the inputs (R22), not from the library
        assert pcpm.pcpm_get_info(h).fixed_point_bits == fb
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


def _hash64(arrs):
    """64-bit digest (blake2b) of the concatenated bytes of a sequence of arrays."""
    import hashlib
    hs = hashlib.blake2b(digest_size=8)
    for a in arrs:
        hs.update(np.ascontiguousarray(a).view(np.uint8))
    return hs.hexdigest()


def _compare_chunked(name, ptr, count, dtype, want, digests, step=1 << 26):
    """GPU array at device `ptr` (count elements) equals want(lo, hi) chunk by chunk
    (bounded host memory at c4 size); records both sides' 64-bit digests."""
    from tests.gpu_util import d2h
    import hashlib
    hg, ho = hashlib.blake2b(digest_size=8), hashlib.blake2b(digest_size=8)
    isz = np.dtype(dtype).itemsize
    for lo in range(0, count, step):
        hi = min(count, lo + step)
        got = d2h(ptr + lo * isz, hi - lo, dtype)
        exp = np.ascontiguousarray(want(lo, hi), dtype=dtype)
        hg.update(got.view(np.uint8))
        ho.update(exp.view(np.uint8))
        if not np.array_equal(got.view(np.uint8), exp.view(np.uint8)):
            bad = lo + int(np.argmax(got != exp))
            raise AssertionError(f"{name}: first difference at element {bad}")
    digests[name] = (hg.hexdigest(), ho.hexdigest())
    assert digests[name][0] == digests[name][1]


@pytest.mark.parametrize("key", ["c3", "c4", "c4bfs", "c5"])
def test_fullsize_layout_matches_oracle(pcpm, key):
    """a0 at the sizes bench.py runs: every layout array of the GPU build (default
    compact layout, the bench's launch configuration) equals the oracle's plain-definition
    layout (oracle.layout) bit for bit -- the 2-byte
    arrays against the oracle's 4-byte bins re-encoded (R20) -- plus the decode anchors
    by their definition and the out-degrees.  Prints per-array 64-bit digests."""
    cfg = graphs.CONFIGS[key]
    b = cfg["bits"]
    g = graphs.make_config(key, backend="torch", device="cuda")
    vals = g.values if key == "c5" else None
    h = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, g.row_ptr, g.col, vals), b, 0,
                           torch.cuda.current_stream())
    gn = g.to_numpy()
    del g
    torch.cuda.empty_cache()
    digests = {}
    try:
        info = pcpm.pcpm_get_info(h)
        v = pcpm.pcpm_export_layout(h)
        ref = oracle.layout(gn.n_src, gn.n_dst, gn.row_ptr, gn.col, b, val=gn.values if key == "c5" else None)
        m, ep, ks, kd = info.nnz, info.e_prime, info.k_src, info.k_dst
        assert (m, ep, ks, kd) == (int(gn.row_ptr[-1]), ref.e_prime, ref.k_src, ref.k_dst)
        qmask = np.uint32((1 << b) - 1)

        def ids16(lo, hi):
            x = ref.ids[lo:hi]
            return ((x & qmask) | ((x >> np.uint32(31)) << np.uint32(15))).astype(np.uint16)
        _compare_chunked("ids16", v.ids16, m, np.uint16, ids16, digests)
        _compare_chunked("png_src16", v.png_src16, ep, np.uint16,
                         lambda lo, hi: (ref.png_src[lo:hi] & qmask).astype(np.uint16), digests)
        flat = lambda a: a.reshape(-1).astype(np.uint32)      # noqa: E731
        for name, arr in [("png_off", flat(ref.png_off)), ("upd_off", flat(ref.upd_off)),
                          ("bin_id_start", flat(ref.bin_id_start)), ("bin_upd_start", flat(ref.bin_upd_start)),
                          ("out_degree", np.diff(gn.row_ptr).astype(np.uint32))]:
            _compare_chunked(name, getattr(v, name), len(arr), np.uint32, lambda lo, hi, a=arr: a[lo:hi], digests)
        if key == "c5":
            _compare_chunked("w", v.w, m, np.float32, lambda lo, hi: ref.w[lo:hi], digests)
        # decode anchors by their plain definition: chunk_base[c] = #flags in ids[0 .. 128 c)
        ncb = m // 128 + 1
        blk = np.zeros(ncb, dtype=np.uint64)          # blk[c + 1] = #flags in ids[128 c .. 128 c + 128)
        step = 1 << 26
        for lo in range(0, (ncb - 1) * 128, step):
            hi = min((ncb - 1) * 128, lo + step)
            blk[1 + lo // 128:1 + hi // 128] = (ref.ids[lo:hi] >> np.uint32(31)).reshape(-1, 128).sum(
                axis=1, dtype=np.uint64)
        cum = np.cumsum(blk).astype(np.uint32)
        _compare_chunked("chunk_base", v.chunk_base, ncb, np.uint32, lambda lo, hi: cum[lo:hi], digests)
    finally:
        pcpm.pcpm_destroy(h)
    print(f"{key}: m={m} E'={ep} k={kd} layout digests (gpu == oracle): "
          + " ".join(f"{k}={d[0]}" for k, d in digests.items()))


def test_fullsize_scatter_bit_exact(pcpm):
    """a1 at c4 size: the scatter of a seeded x through the bench's layout equals the
    oracle's Alg. 4 copy (oracle.scatter on the oracle layout) bit for bit."""
    key = "c4"
    cfg = graphs.CONFIGS[key]
    g = graphs.make_config(key, backend="torch", device="cuda")
    h = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, g.row_ptr, g.col, None), cfg["bits"], 0,
                           torch.cuda.current_stream())
    gn = g.to_numpy()
    del g
    torch.cuda.empty_cache()
    digests = {}
    try:
        x = np.random.default_rng(7).random(gn.n_src).astype(np.float32)
        pcpm.pcpm_scatter(h, torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        info = pcpm.pcpm_get_info(h)
        v = pcpm.pcpm_export_layout(h)
        ref = oracle.scatter(oracle.layout(gn.n_src, gn.n_dst, gn.row_ptr, gn.col, cfg["bits"]), x)
        assert len(ref) == info.e_prime
        _compare_chunked("upd", v.upd, info.e_prime, np.uint32, lambda lo, hi: ref[lo:hi].view(np.uint32), digests)
    finally:
        pcpm.pcpm_destroy(h)
    print(f"{key}: scatter of E'={info.e_prime} updates bit-exact, digest {digests['upd'][0]}")


def test_fullsize_pair_q16_bit_identical_to_q15(pcpm):
    """q = 2^16 (pair handles) at c3's size: the fixed-point sums are exact and order-free and the
    apply is the same arithmetic, so the output must equal the b = 15 handle's (which
    test_fullsize_pagerank compares with the oracle) bit for bit; r must not fall."""
    key = "c3"
    cfg = graphs.CONFIGS[key]
    g = graphs.make_config(key, backend="torch", device="cuda")
    outs, eps = [], []
    for b in (15, 16):
        h = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, g.row_ptr, g.col, None), b, 0,
                               torch.cuda.current_stream())
        try:
            info = pcpm.pcpm_get_info(h)
            assert info.partition_bits == b and info.k_dst == (g.n_dst + (1 << b) - 1) >> b
            out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
            pcpm.pcpm_pagerank(h, 0.85, cfg["iters"], out)
            torch.cuda.synchronize()
            outs.append(out)
            eps.append(info.e_prime)
        finally:
            pcpm.pcpm_destroy(h)
    assert torch.equal(outs[0], outs[1])
    assert eps[1] <= eps[0]                       # larger partitions compress more
    assert abs(float(outs[1].double().sum()) - 1.0) <= 1e-5
