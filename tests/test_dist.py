"""Multi-GPU path: destination shards + all-gather, on CPU with gloo.

The per-shard compute is libpcpm.so on a GPU; here a test-side step (fp64
Eq. 1 on the shard's vertices, fp32 storage like the kernels) stands in for it,
so these tests check the decomposition and the exchange: shard bounds, padded
all-gather of SPR slices, all-reduce of (residual, dangling mass), and that the
assembled vector equals the unsharded oracle.  world_size 2 over gloo on
127.0.0.1.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from inputs import graphs
from paper_1709_07122_b200 import dist as pdist


def test_shard_plan_covers_vertices_in_whole_partitions():
    for n, b, world in [(1000, 4, 2), (4096, 8, 3), (70001, 10, 8), (5, 3, 4), (1 << 20, 15, 8)]:
        plan = pdist.shard_plan(n, b, world)
        assert plan.per % (1 << b) == 0
        edges = [plan.bounds(r) for r in range(world)]
        assert edges[0][0] == 0 and edges[-1][1] == n
        for (lo, hi), (lo2, _) in zip(edges, edges[1:]):
            assert hi == lo2 and lo <= hi
        assert plan.padded >= n


class OracleStep:
    """Test stand-in for pcpm_shard_init / pcpm_shard_step (Eq. 1 with R1, fp64 math, fp32 storage)."""

    def __init__(self, n, row_ptr, col):
        self.n = n
        self.deg = np.diff(row_ptr)
        self.in_ptr, self.in_src = oracle.transpose(n, row_ptr, col)

    def init(self, sh, pr0, spr0, dang0):
        lo, hi = sh.lo, sh.hi
        pr0[:] = torch.tensor(np.full(hi - lo, 1.0 / self.n), dtype=torch.float32)
        dg = self.deg[lo:hi]
        spr0[:] = torch.tensor(np.where(dg > 0, (1.0 / self.n) / np.maximum(dg, 1), 0.0), dtype=torch.float32)
        dang0[0] = float(np.count_nonzero(dg == 0)) / self.n

    def step(self, sh, d, spr_in, D_in, pr_old, pr_new, spr_out, red_out):
        lo, hi, n = sh.lo, sh.hi, self.n
        spr = spr_in[:n].numpy().astype(np.float64)
        D = float(D_in[0])
        new = np.empty(hi - lo)
        for i, v in enumerate(range(lo, hi)):
            s = spr[self.in_src[self.in_ptr[v]:self.in_ptr[v + 1]]].sum()
            new[i] = (1.0 - d) / n + d * (s + D / n)
        dg = self.deg[lo:hi]
        pr_new[:hi - lo] = torch.tensor(new, dtype=torch.float32)
        spr_out[:hi - lo] = torch.tensor(np.where(dg > 0, new / np.maximum(dg, 1), 0.0), dtype=torch.float32)
        red_out[0] = float(np.abs(new - pr_old[:hi - lo].numpy().astype(np.float64)).sum())
        red_out[1] = float(new[dg == 0].sum())


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = graphs.make_graph("rmat", 21, scale=11, permute=True)
        sh = pdist.ShardedPageRank(g.n_src, g.row_ptr, g.col, 6, device="cpu",
                                   step_impl=OracleStep(g.n_src, g.row_ptr, g.col))
        pr = sh.run(0.85, 12)
        full = sh.gather_pr(pr).numpy()
        res = [float(r) for r in sh.residuals]
        q.put((rank, sh.lo, sh.hi, full, res))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sharded_pagerank_gloo_matches_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = graphs.make_graph("rmat", 21, scale=11, permute=True)
    ref = oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, 12)
    out.sort()
    assert out[0][1] == 0 and out[-1][2] == g.n_src and out[0][2] == out[1][1]
    for _, _, _, full, res in out:
        rel = np.abs(full.astype(np.float64) - ref) / ref
        assert rel.max() <= 1e-5 and np.abs(full - ref).sum() <= 1e-6
        # the all-reduced residual is the global L1 change, identical on every rank
        np.testing.assert_allclose(res, out[0][4])
    prs = [oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, t) for t in range(13)]
    want = [np.abs(prs[t + 1] - prs[t]).sum() for t in range(12)]
    np.testing.assert_allclose(out[0][4], want, rtol=1e-4, atol=1e-7)


class FakeIpc:
    """Stand-in for the CUDA IPC calls of libpcpm (pcpm_ipc_*): integer 'pointers'."""

    def __init__(self, rank, fail_open):
        self.rank, self.fail_open = rank, fail_open
        self.freed, self.closed, self.next = [], [], (rank + 1) << 40

    def pcpm_ipc_alloc(self, nbytes):
        self.next += 1 << 30
        return self.next

    def pcpm_ipc_get_handle(self, ptr):
        return ptr.to_bytes(8, "little") * 8

    def pcpm_ipc_open(self, handle):
        if self.fail_open:
            raise RuntimeError("no peer access")
        return int.from_bytes(handle[:8], "little") + 7      # a mapping in this process

    def pcpm_ipc_close(self, ptr):
        self.closed.append(ptr)

    def pcpm_ipc_free(self, ptr):
        self.freed.append(ptr)


def _p2p_worker(rank, world, port, q, fail_rank):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = object.__new__(pdist.ShardedPageRank)
    sh.torch, sh.dist, sh.group, sh.device = torch, dist, None, "cpu"
    sh.world, sh.rank = world, rank
    sh.plan = pdist.shard_plan(5000, 8, world)
    sh.exchange, sh.exchange_note, sh.own, sh.peers = "p2p", "", None, None
    sh.pcpm = FakeIpc(rank, fail_open=(rank == fail_rank))
    sh._setup_p2p()
    res = {"exchange": sh.exchange, "note": sh.exchange_note, "freed": len(sh.pcpm.freed),
           "closed": len(sh.pcpm.closed)}
    if sh.exchange == "p2p":
        outs = sh._outs(1)
        off = rank * sh.plan.per * 4
        res["outs_ok"] = outs[0] == sh.own[1] + off and len(outs) == world and \
            all(o == sh.peers[r][1] + off for o, r in zip(outs[1:], sorted(sh.peers)))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, res))


@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_p2p_exchange_setup_is_consistent_across_ranks(fail_rank):
    """The fused-exchange setup (IPC handles exchanged once, peers mapped) either
    succeeds on every rank or falls back to the NCCL all-gather on every rank (a
    rank that cannot map a peer must not leave the others waiting)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q, fail_rank)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, res in out.items():
        if fail_rank < 0:
            assert res["exchange"] == "p2p" and res["outs_ok"] and res["freed"] == 0
        else:
            assert res["exchange"] == "allgather" and "p2p setup failed" in res["note"]
            assert res["freed"] == 2                       # own exchange buffers released
            assert res["closed"] == (0 if r == fail_rank else 2 * (world - 1))
