"""Destination shards on one GPU (the per-rank compute of the multi-GPU path).

All shard handles live in one process on cuda:0 and write their SPR slices into
one shared full vector, so no rank waits on another; the exchange itself is
covered by tests/test_dist.py (gloo).  Checks: each shard's layout is
bit-exact against the oracle layout of its column slice; N shards reproduce the
oracle PageRank within the BASELINE bounds; one shard is bit-identical to
pcpm_pagerank (same kernels, same reduction order).
"""
import numpy as np
import pytest

import oracle
from inputs import graphs
from paper_1709_07122_b200 import dist as pdist
from tests.gpu_util import d2h, to_device

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pcpm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1709_07122_b200 import pcpm as p
    return p


def column_slice(g, lo, hi):
    rows = np.repeat(np.arange(g.n_src), np.diff(g.row_ptr))
    keep = (g.col >= lo) & (g.col < hi)
    rp = np.zeros(g.n_src + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=g.n_src), out=rp[1:])
    return rp, (g.col[keep] - lo).astype(np.uint32)


def run_shards(pcpm, g, b, nsh, d, iters):
    plan = pdist.shard_plan(g.n_src, b, nsh)
    rp, col, _ = to_device(g)
    csr = pcpm.make_csr(g.n_src, g.n_dst, rp, col, None)
    hs = [pcpm.pcpm_build_shard(csr, b, *plan.bounds(r)) for r in range(nsh)]
    try:
        f32 = dict(dtype=torch.float32, device="cuda")
        spr = [torch.zeros(plan.padded + 8, **f32), torch.zeros(plan.padded + 8, **f32)]
        n_loc = [hi - lo for lo, hi in (plan.bounds(r) for r in range(nsh))]
        pr = [[torch.zeros(max(nl, 1), **f32), torch.zeros(max(nl, 1), **f32)] for nl in n_loc]
        red = torch.zeros(nsh, 2, dtype=torch.float64, device="cuda")
        D = torch.zeros(1, dtype=torch.float64, device="cuda")
        chunk = lambda buf, r: buf[r * plan.per:(r + 1) * plan.per]     # noqa: E731
        for r, h in enumerate(hs):
            pcpm.pcpm_shard_init(h, pr[r][0], chunk(spr[0], r), red[r, 1:])
        D.copy_(red[:, 1].sum().reshape(1))
        for t in range(iters):
            cur, nxt = t & 1, (t + 1) & 1
            for r, h in enumerate(hs):
                pcpm.pcpm_shard_step(h, d, spr[cur], D, pr[r][cur], pr[r][nxt], chunk(spr[nxt], r), red[r])
            D.copy_(red[:, 1].sum().reshape(1))
        torch.cuda.synchronize()
        full = torch.cat([pr[r][iters & 1][:n_loc[r]] for r in range(nsh)]).cpu().numpy()
        return full, hs, plan
    except Exception:
        for h in hs:
            pcpm.pcpm_destroy(h)
        raise


@pytest.mark.parametrize("nsh", [1, 2, 3])
def test_shards_match_oracle(pcpm, nsh):
    g = graphs.make_graph("rmat", 31, scale=14, permute=True)
    b, d, iters = 9, 0.85, 15
    full, hs, plan = run_shards(pcpm, g, b, nsh, d, iters)
    try:
        ref = oracle.pagerank(g.n_src, g.row_ptr, g.col, d, iters)
        rel = np.abs(full.astype(np.float64) - ref) / ref
        assert rel.max() <= 1e-5 and np.abs(full - ref).sum() <= 1e-6
        # each shard's bins = the oracle layout of its column slice (bit-exact)
        for r, h in enumerate(hs):
            lo, hi = plan.bounds(r)
            srp, scol = column_slice(g, lo, hi)
            lay = oracle.layout(g.n_src, hi - lo, srp, scol, b)
            info = pcpm.pcpm_get_info(h)
            v = pcpm.pcpm_export_layout(h)
            assert info.e_prime == lay.e_prime and info.nnz == len(scol)
            ids = lay.ids
            want16 = ((ids & np.uint32((1 << b) - 1)) | ((ids >> np.uint32(31)) << np.uint32(15))).astype(np.uint16)
            np.testing.assert_array_equal(d2h(v.ids16, info.nnz, np.uint16), want16)
            np.testing.assert_array_equal(d2h(v.png_src16, info.e_prime, np.uint16),
                                          (lay.png_src & np.uint32((1 << b) - 1)).astype(np.uint16))
            # global out-degrees are kept (the slice's rows only hold edges into the slice)
            np.testing.assert_array_equal(d2h(v.out_degree, g.n_src, np.uint32), np.diff(g.row_ptr))
        if nsh == 1:
            out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
            rp, col, _ = to_device(g)
            h1 = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, rp, col, None), b, 0, None)
            try:
                pcpm.pcpm_pagerank(h1, d, iters, out)
                np.testing.assert_array_equal(out.cpu().numpy(), full)
            finally:
                pcpm.pcpm_destroy(h1)
    finally:
        for h in hs:
            pcpm.pcpm_destroy(h)


def test_shard_arguments_rejected(pcpm):
    g = graphs.make_graph("rmat", 31, scale=10, permute=True)
    rp, col, _ = to_device(g)
    csr = pcpm.make_csr(g.n_src, g.n_dst, rp, col, None)
    for lo, hi in [(-1, 10), (10, 5), (0, g.n_src + 1), (3, 64)]:   # v_lo must be a multiple of q
        with pytest.raises(pcpm.PcpmError):
            pcpm.pcpm_build_shard(csr, 5, lo, hi)


def run_shards_fused(pcpm, g, b, nsh, d, iters):
    """Each shard owns its own full-SPR buffers (as each rank would); its step stores
    its SPR slice into every shard's buffer (pcpm_shard_step_peers, the fused
    exchange) -- here all buffers are on one GPU and the shards run one after
    another, so no shard waits on another."""
    plan = pdist.shard_plan(g.n_src, b, nsh)
    rp, col, _ = to_device(g)
    csr = pcpm.make_csr(g.n_src, g.n_dst, rp, col, None)
    hs = [pcpm.pcpm_build_shard(csr, b, *plan.bounds(r)) for r in range(nsh)]
    try:
        f32 = dict(dtype=torch.float32, device="cuda")
        spr = [[torch.zeros(plan.padded + 8, **f32), torch.zeros(plan.padded + 8, **f32)] for _ in range(nsh)]
        n_loc = [hi - lo for lo, hi in (plan.bounds(r) for r in range(nsh))]
        pr = [[torch.zeros(max(nl, 1), **f32), torch.zeros(max(nl, 1), **f32)] for nl in n_loc]
        red = torch.zeros(nsh, 2, dtype=torch.float64, device="cuda")
        D = torch.zeros(1, dtype=torch.float64, device="cuda")
        chunk = lambda buf, r: buf[r * plan.per:(r + 1) * plan.per]     # noqa: E731
        for r, h in enumerate(hs):
            outs = [chunk(spr[r][0], r)] + [chunk(spr[s][0], r) for s in range(nsh) if s != r]
            pcpm.pcpm_shard_init_peers(h, pr[r][0], outs, red[r, 1:])
        D.copy_(red[:, 1].sum().reshape(1))
        for t in range(iters):
            cur, nxt = t & 1, (t + 1) & 1
            for r, h in enumerate(hs):
                outs = [chunk(spr[r][nxt], r)] + [chunk(spr[s][nxt], r) for s in range(nsh) if s != r]
                pcpm.pcpm_shard_step_peers(h, d, spr[r][cur], D, pr[r][cur], pr[r][nxt], outs, red[r])
            D.copy_(red[:, 1].sum().reshape(1))
        torch.cuda.synchronize()
        for s in range(1, nsh):                         # every rank holds the same full SPR vector
            assert torch.equal(spr[s][iters & 1][:g.n_src], spr[0][iters & 1][:g.n_src])
        full = torch.cat([pr[r][iters & 1][:n_loc[r]] for r in range(nsh)]).cpu().numpy()
        return full
    finally:
        for h in hs:
            pcpm.pcpm_destroy(h)


@pytest.mark.parametrize("case", ["rmat14_b9", "er_ragged_b10"])
@pytest.mark.parametrize("nsh", [2, 3])
def test_fused_exchange_matches_allgather_and_oracle(pcpm, nsh, case):
    if case == "rmat14_b9":
        g, b = graphs.make_graph("rmat", 31, scale=14, permute=True), 9
    else:                                               # n % 4 != 0: scalar apply path, split bins
        g, b = graphs.make_graph("er", 6, n=70001, m_raw=600000), 10
    d, iters = 0.85, 12
    fused = run_shards_fused(pcpm, g, b, nsh, d, iters)
    ref = oracle.pagerank(g.n_src, g.row_ptr, g.col, d, iters)
    rel = np.abs(fused.astype(np.float64) - ref) / ref
    assert rel.max() <= 1e-5 and np.abs(fused - ref).sum() <= 1e-6
    shared, hs, _ = run_shards(pcpm, g, b, nsh, d, iters)
    for h in hs:
        pcpm.pcpm_destroy(h)
    np.testing.assert_array_equal(fused, shared)      # same kernels, same sums: bit-identical


def test_peer_step_arguments_and_ipc_buffers(pcpm):
    g = graphs.make_graph("rmat", 31, scale=10, permute=True)
    rp, col, _ = to_device(g)
    h = pcpm.pcpm_build_shard(pcpm.make_csr(g.n_src, g.n_dst, rp, col, None), 6, 0, g.n_src)
    try:
        f = torch.zeros(g.n_src + 8, dtype=torch.float32, device="cuda")
        red = torch.zeros(2, dtype=torch.float64, device="cuda")
        D = torch.zeros(1, dtype=torch.float64, device="cuda")
        for outs in ([], [f] * (pcpm.PCPM_MAX_PEERS + 2)):
            with pytest.raises(pcpm.PcpmError) as e:
                pcpm.pcpm_shard_step_peers(h, 0.85, f, D, f, f, outs, red)
            assert e.value.code == pcpm.PCPM_EINVAL
        with pytest.raises(pcpm.PcpmError):
            pcpm.pcpm_shard_step_peers(h, 0.85, f, D, f, f, [f, np.zeros(4, np.float32)], red)   # host peer
    finally:
        pcpm.pcpm_destroy(h)
    ptr = pcpm.pcpm_ipc_alloc(1 << 20)
    try:
        assert len(pcpm.pcpm_ipc_get_handle(ptr)) == 64
    finally:
        pcpm.pcpm_ipc_free(ptr)
