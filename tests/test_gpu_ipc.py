"""The fused multi-GPU exchange across PROCESSES, on one GPU.

Two ranks (torch.multiprocessing spawn, gloo collectives, both on cuda:0) run
paper_1709_07122_b200.dist.ShardedPageRank with exchange="p2p": each rank builds its
destination shard (pcpm_build_shard), allocates its two full-SPR exchange buffers
(pcpm_ipc_alloc), exchanges their CUDA IPC handles (all_gather_object) and maps the
other process's buffers (pcpm_ipc_open, a real cudaIpcOpenMemHandle in another
process); every iteration's gather (pcpm_shard_step_peers) stores the rank's SPR
slice into BOTH processes' buffers, and the 16-byte all-reduce orders the next
iteration after the peer's stores.  No kernel waits on another rank's kernel: the
only cross-rank ordering is the host-side collective, so the two processes may
share one GPU.  The gathered PR must match the fp64 oracle within the north-star
bounds, and every rank must see the same per-iteration residuals.
"""
import os
import socket

import numpy as np
import pytest

import oracle
from inputs import graphs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ITERS = 12
B = 9


def _graph():
    return graphs.make_graph("rmat", 31, scale=14, permute=True)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1709_07122_b200 import dist as pdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        g = _graph()
        rp = torch.from_numpy(g.row_ptr).cuda()
        col = torch.from_numpy(g.col.view(np.int32)).cuda()
        sh = pdist.ShardedPageRank(g.n_src, rp, col, B, device="cuda", exchange="p2p")
        try:
            pr = sh.run(0.85, ITERS)
            torch.cuda.synchronize()
            res = [float(r) for r in sh.residuals]
            q.put((rank, sh.lo, sh.hi, sh.exchange, sh.exchange_note, pr.cpu().numpy(), res))
        finally:
            sh.close()
    except Exception as e:                     # noqa: BLE001 -- reported to the parent
        q.put((rank, -1, -1, "error", repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_fused_exchange_across_processes_matches_oracle():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for rank, lo, hi, ex, note, _, _ in out:
        assert ex == "p2p", f"rank {rank}: exchange {ex} ({note})"
    assert all(p.exitcode == 0 for p in procs)
    g = _graph()
    ref = oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, ITERS)
    assert out[0][1] == 0 and out[-1][2] == g.n_src and out[0][2] == out[1][1]
    full = np.concatenate([o[5][:o[2] - o[1]] for o in out]).astype(np.float64)
    rel = np.abs(full - ref) / ref
    assert rel.max() <= 1e-5 and np.abs(full - ref).sum() <= 1e-6, (rel.max(), np.abs(full - ref).sum())
    np.testing.assert_array_equal(out[0][6], out[1][6])          # the all-reduced residuals agree
    prs = [oracle.pagerank(g.n_src, g.row_ptr, g.col, 0.85, t) for t in range(ITERS + 1)]
    want = [np.abs(prs[t + 1] - prs[t]).sum() for t in range(ITERS)]
    np.testing.assert_allclose(out[0][6], want, rtol=1e-4, atol=1e-7)
