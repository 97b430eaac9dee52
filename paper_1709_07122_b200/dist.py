"""Multi-GPU PCPM PageRank: destination shards + one all-gather per iteration.

SURVEY §8(e) / DESIGN.md §7.  Rank r of N owns the destination vertices
[lo_r, hi_r): whole partitions of q = 2^b vertices, ceil(k / N) per rank.  Its
handle (pcpm_build_shard) holds the bins of those partitions only, built from
the column slice of the full CSR, with the global out-degrees.  One iteration
on every rank:

  1. pcpm_shard_step: scatter all source partitions into its own bins (Alg. 4),
     gather + apply its vertices (Alg. 5 + Eq. 1), writing SPR_{t+1} of its
     slice straight into its chunk of the next full-SPR buffer;
  2. all_gather_into_tensor of the SPR chunks (n * 4 bytes in all; NCCL over
     NVLink/NVSwitch on B200) -- the only data-path exchange;
  3. all_reduce of (residual, dangling mass), 16 bytes, for D_{t+1}.

The full-SPR buffers are padded to N equal chunks of ceil(k/N) * q floats so
the gathered vector is contiguous in global vertex order.

exchange="p2p" fuses step 2 into step 1: every rank's full-SPR buffers are plain
cudaMalloc allocations whose CUDA IPC handles are exchanged once; the gather's
apply then stores each SPR group of the slice into every rank's buffer directly
(pcpm_shard_step_peers, NVLink P2P stores overlapping the gather), and the
16-byte all-reduce of step 3 orders the ranks' next iteration after all stores
(each gather ends with a system-scope fence).  This module is
plumbing (torch.distributed + device buffers); all arithmetic of the method
runs in libpcpm.so.  ``step_impl`` lets the CPU tests (gloo, world_size 2)
drive the same exchange with a test-side per-shard step.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class ShardPlan:
    n: int
    b: int
    world: int
    per: int          # vertices per chunk (a multiple of q)

    @property
    def padded(self) -> int:
        return self.per * self.world

    def bounds(self, rank: int):
        lo = min(self.n, rank * self.per)
        hi = min(self.n, (rank + 1) * self.per)
        return lo, hi


def shard_plan(n: int, b: int, world: int) -> ShardPlan:
    """Equal whole-partition chunks: rank r owns partitions [r*pk, (r+1)*pk), pk = ceil(k/N)."""
    q = 1 << b
    k = (n + q - 1) // q
    pk = (k + world - 1) // world
    return ShardPlan(n=n, b=b, world=world, per=pk * q)


class ShardedPageRank:
    """PCPM PageRank of one graph over the ranks of a torch.distributed group.

    row_ptr / col: the full CSR (every rank passes the same graph; only the
    column slice of this rank is kept on its device after the build).
    """

    def __init__(self, n, row_ptr, col, b, group=None, device=None, stream=None, step_impl=None, timing=False,
                 exchange="allgather"):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.plan = shard_plan(n, b, self.world)
        self.lo, self.hi = self.plan.bounds(self.rank)
        self.n, self.b = n, b
        self.device = device
        self.h = None
        self.step_impl = step_impl
        if step_impl is None:
            from . import pcpm
            self.pcpm = pcpm
            if self.hi > self.lo:
                csr = pcpm.make_csr(n, n, row_ptr, col, None)
                self.h = pcpm.pcpm_build_shard(csr, b, self.lo, self.hi, 0, stream)
        n_loc = max(self.hi - self.lo, 0)
        f32 = dict(dtype=torch.float32, device=device)
        self.spr = [torch.zeros(self.plan.padded + 8, **f32), torch.zeros(self.plan.padded + 8, **f32)]
        self.pr = [torch.zeros(max(n_loc, 1), **f32), torch.zeros(max(n_loc, 1), **f32)]
        self.red = torch.zeros(2, dtype=torch.float64, device=device)     # residual, dangling mass
        self.D = torch.zeros(1, dtype=torch.float64, device=device)
        self.residuals = []
        self.timing = timing and step_impl is None
        self.events = []          # per iteration: (before step, after step, after exchange)
        self.exchange = exchange if (step_impl is None and self.world > 1) else "allgather"
        self.exchange_note = ""
        self.own = self.peers = None
        if self.exchange == "p2p":
            self._setup_p2p()

    def _setup_p2p(self):
        """Own full-SPR buffers (cudaMalloc, IPC-shareable) and the peers' buffers opened here.
        If any rank cannot map a peer (no P2P path), every rank falls back to the all-gather."""
        pc = self.pcpm
        nbytes = (self.plan.padded + 8) * 4
        ok, why = 1, ""
        mine = None
        try:
            self.own = [pc.pcpm_ipc_alloc(nbytes), pc.pcpm_ipc_alloc(nbytes)]
            mine = [pc.pcpm_ipc_get_handle(p) for p in self.own]
        except Exception as e:               # noqa: BLE001 -- reported through self.exchange_note
            ok, why = 0, str(e)
        every = [None] * self.world
        self.dist.all_gather_object(every, mine, group=self.group)
        self.peers = {}
        if ok and all(h is not None for h in every):
            try:
                for r in range(self.world):
                    if r != self.rank:
                        self.peers[r] = [pc.pcpm_ipc_open(hd) for hd in every[r]]
            except Exception as e:           # noqa: BLE001
                ok, why = 0, str(e)
        else:
            ok = 0
        flag = self.torch.tensor([ok], dtype=self.torch.int32, device=self.device)
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=self.group)
        if int(flag.item()) == 0:            # consistent fallback on every rank
            for ptrs in self.peers.values():
                for p in ptrs:
                    pc.pcpm_ipc_close(p)
            self.dist.barrier(group=self.group)
            for p in self.own or []:
                pc.pcpm_ipc_free(p)
            self.own, self.peers = None, None
            self.exchange = "allgather"
            self.exchange_note = "p2p setup failed (" + (why or "on another rank") + "); NCCL all-gather"
        self.dist.barrier(group=self.group)

    def _outs(self, buf):
        """This rank's chunk in its own buffer, then in every peer's (buf = 0 or 1)."""
        off = self.rank * self.plan.per * 4
        return [self.own[buf] + off] + [self.peers[r][buf] + off for r in sorted(self.peers)]

    def info(self):
        return self.pcpm.pcpm_get_info(self.h) if self.h is not None else None

    def phase_ms(self):
        """(compute ms, exchange ms) summed over the iterations of the last run (device events)."""
        self.torch.cuda.synchronize()
        comp = sum(a.elapsed_time(b) for a, b, _ in self.events)
        comm = sum(b.elapsed_time(c) for _, b, c in self.events)
        return comp, comm

    def _event(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def close(self):
        if self.h is not None:
            self.pcpm.pcpm_destroy(self.h)
            self.h = None
        if self.peers:
            self.torch.cuda.synchronize()
            self.dist.barrier(group=self.group)          # no peer still writes into our buffers
            for ptrs in self.peers.values():
                for p in ptrs:
                    self.pcpm.pcpm_ipc_close(p)
            self.peers = None
        if self.own:
            self.dist.barrier(group=self.group)          # every peer closed its mapping first
            for p in self.own:
                self.pcpm.pcpm_ipc_free(p)
            self.own = None

    def _chunk(self, buf):
        return buf[self.rank * self.plan.per:(self.rank + 1) * self.plan.per]

    def _allgather(self, buf):
        if self.world > 1:
            self.dist.all_gather_into_tensor(buf[:self.plan.padded], self._chunk(buf).clone()
                                             if buf.device.type == "cpu" else self._chunk(buf), group=self.group)

    def _allreduce(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, group=self.group)

    def run(self, d: float = 0.85, iters: int = 20):
        """PR_iters of this rank's slice (device f32[hi - lo]); residuals in self.residuals."""
        n_loc = self.hi - self.lo
        # PR_0 = 1/n, SPR_0, D_0 (R2, R1)
        self.red.zero_()
        p2p = self.exchange == "p2p"
        if n_loc > 0:
            if p2p:
                self.pcpm.pcpm_shard_init_peers(self.h, self.pr[0], self._outs(0), self.red[1:])
            elif self.step_impl is None:
                self.pcpm.pcpm_shard_init(self.h, self.pr[0], self._chunk(self.spr[0]), self.red[1:])
            else:
                self.step_impl.init(self, self.pr[0][:n_loc], self._chunk(self.spr[0])[:n_loc], self.red[1:])
        if not p2p:
            self._allgather(self.spr[0])
        self.D.copy_(self.red[1:])
        self._allreduce(self.D)
        self.residuals = []
        self.events = []
        for t in range(iters):
            cur, nxt = t & 1, (t + 1) & 1
            self.red.zero_()
            ev = [self._event()] if self.timing else None
            if n_loc > 0:
                if p2p:                                     # SPR_{t+1} stored to every rank by the apply
                    self.pcpm.pcpm_shard_step_peers(self.h, d, self.own[cur], self.D, self.pr[cur], self.pr[nxt],
                                                    self._outs(nxt), self.red)
                else:
                    args = (d, self.spr[cur], self.D, self.pr[cur], self.pr[nxt], self._chunk(self.spr[nxt]),
                            self.red)
                    if self.step_impl is None:
                        self.pcpm.pcpm_shard_step(self.h, *args)
                    else:
                        self.step_impl.step(self, *args)
            if ev:
                ev.append(self._event())
            if not p2p:
                self._allgather(self.spr[nxt])             # SPR_{t+1} of all vertices
            self._allreduce(self.red)                       # global residual and D_{t+1} (p2p: also the
                                                            # barrier after every rank's stores)
            if ev:
                ev.append(self._event())
                self.events.append(tuple(ev))
            self.D.copy_(self.red[1:])
            self.residuals.append(self.red[0].clone())
        return self.pr[iters & 1][:n_loc]

    def gather_pr(self, pr_slice):
        """Full PR vector on every rank (test / output helper)."""
        torch = self.torch
        buf = torch.zeros(self.plan.padded, dtype=torch.float32, device=pr_slice.device)
        n_loc = self.hi - self.lo
        self._chunk(buf)[:n_loc].copy_(pr_slice[:n_loc])
        self._allgather(buf)
        return buf[:self.n]
