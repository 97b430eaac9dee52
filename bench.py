#!/usr/bin/env python
"""bench.py -- GTEPS per PageRank iteration and achieved HBM GB/s of the PCPM hot
path on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl pcpm|reference]

A step is one pcpm_pagerank call of the config's iteration count (20 for
RMAT-26: scatter -> gather+apply per iteration, §5 protocol P:436)
on the device-resident layout; value = m * iters * K * N / max-over-ranks time
(GTEPS, the paper's "giga edges / runtime of a single iteration").
The SpMV config (c5) steps 50 multiplies and reports G-nonzeros/s.
Multi-GPU runs independent replicas (the single-graph path is not
sharded in this round), so scaling is weak.

--impl reference times the CPU oracle (oracle/, fp64 C, OpenMP) on the host
cores on a bounded sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "GTEPS per PageRank iteration and achieved HBM GB/s (% of peak) on 1 B200"
WORKLOADS = {
    "c1": "c1_rmat10: RMAT scale 10 ef16 seed1 (a,b,c)=(.57,.19,.19) unpermuted, q=2^8, d=0.85, 10 iterations",
    "c2": "c2_er20: Erdos-Renyi 2^20 vertices 2^24 raw edges seed2, q=2^15, d=0.85, 20 iterations",
    "c3": "c3_rmat24: RMAT scale 24 ef16 seed3 random labels, q=2^15, d=0.85, 20 iterations",
    "c4": "c4_rmat26: RMAT scale 26 ef16 seed4 random labels, q=2^15, d=0.85, 20 iterations",
    "c4bfs": "c4_rmat26_bfs: c4's graph relabelled in BFS order from the highest-out-degree vertex (R16), "
             "q=2^15, d=0.85, 20 iterations",
    "c5": "c5_spmv_rmat25: y=A.x, RMAT scale 25 ef16 seed5 random labels, values/x U[-1,1), q=2^15, 50 multiplies",
    "c4w": "c4w_rmat26_weighted: weighted PageRank (P:287-288, R24) on c4's graph, weights |U[-1,1)| per raw edge, "
           "q=2^15, d=0.85, 20 iterations",
    "c5ns": "c5ns_spmv_rmat25_2to1: non-square y=M^T x, c5's matrix restricted to its first 2^24 columns "
            "(2^25 x 2^24), q=2^15, 50 multiplies",
}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            out = self.p.communicate(timeout=5)[0]
        except Exception:
            self.p.kill()
            return None
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def make_graph(key, device):
    from inputs import graphs
    return graphs.make_config(key, backend="torch", device=device)


def layout_bytes(info, iters_kind="pagerank", wide=False, weighted=False):
    """Algorithmic bytes per launch of each kernel.

    d_i = 2 (compact layout: 2-byte IDs and PNG sources) or 4 (PCPM_WIDE_IDS), d_v = 4.
    """
    n, m, ep, ks, kd = info.n_src, info.nnz, info.e_prime, info.k_src, info.k_dst
    di = 4 if wide else 2
    scatter = di * ep + 4 * ep + 4 * n + 4 * ks * (kd + 1) + 4 * ks * kd
    if iters_kind == "pagerank":
        gather = di * m + 4 * ep + 4 * n * 4      # ids, updates; outdeg + PR_old read, PR + SPR written
        if weighted:
            gather += 4 * m                       # weighted PageRank (R24): the weights beside the IDs
    else:
        gather = di * m + 4 * m + 4 * ep + 4 * info.n_dst   # ids, weights, updates; y written
    if getattr(info, "compact_slots", 0):
        gather += 2 * info.n_dst                   # the apply reads each vertex's accumulator slot
    return scatter, gather


def build_bytes(info, weighted=False):
    """Algorithmic bytes of the counting build (DESIGN.md §5 "build"; the Table 8 analogue):
    two passes over the CSR (row_ptr 8(n+1) + col 4m each, + values 4m in the second),
    out-degrees and 1/out-degree written (8n), the IDs (2m) and PNG sources (2E') placed,
    the IDs re-read for the decode anchors (2m)."""
    n, m, ep = info.n_src, info.nnz, info.e_prime
    return 2 * (8 * (n + 1) + 4 * m) + (4 * m if weighted else 0) + 8 * n + 2 * m + 2 * ep + 2 * m + \
        (4 * m if weighted else 0)


# ---------------------------------------------------------------------------- PCPM arm


def run_pcpm(args, world, rank, local):
    import torch
    from paper_1709_07122_b200 import model, pcpm

    key = args.config
    dev = torch.device("cuda", local)
    g = make_graph(key, dev)
    cfg = g.meta
    op = cfg["op"]
    iters = args.iters or cfg["iters"]
    b = args.bits or cfg["bits"]
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    csr = pcpm.make_csr(g.n_src, g.n_dst, g.row_ptr, g.col, g.values)
    weighted_pr = op == "pagerank" and g.values is not None       # c4w: weighted PageRank (R24)
    flags = 0
    if args.wide:
        flags |= pcpm.PCPM_WIDE_IDS
    if args.no_compress:
        flags |= pcpm.PCPM_NO_COMPRESS
    if args.slots:
        flags |= pcpm.PCPM_COMPACT_SLOTS
    if args.engine == "bvgas":
        flags |= pcpm.PCPM_BVGAS                  # the BVGAS comparison engine (Alg. 3)
    # the first build grows the stream-ordered memory pool; build_ms is the median of the next three
    h = pcpm.pcpm_build_ex(csr, b, flags, stream)
    build_ms_cold = pcpm.pcpm_get_info(h).build_ms
    bms = []
    for _ in range(3):
        pcpm.pcpm_destroy(h)
        h = pcpm.pcpm_build_ex(csr, b, flags, stream)
        bms.append(pcpm.pcpm_get_info(h).build_ms)
    build_ms = statistics.median(bms)
    info = pcpm.pcpm_get_info(h)
    m, n = info.nnz, info.n_src
    if weighted_pr:
        pcpm.pcpm_set_option(h, "weighted_pagerank", 1)
    for kv in args.opt:                   # kernel-variant A/B experiments
        k, v = kv.split("=")
        pcpm.pcpm_set_option(h, k, int(v))
    out = torch.zeros(max(g.n_src, g.n_dst), dtype=torch.float32, device=dev)

    if op == "pagerank":
        def step():
            pcpm.pcpm_pagerank(h, 0.85, iters, out)
        units_per_step = m * iters
    else:
        from inputs import graphs
        x = graphs.make_x(g.n_src, cfg["seed"], backend="torch", device=dev)

        def step():
            for _ in range(iters):
                pcpm.pcpm_spmv(h, x, out)
        units_per_step = m * iters

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    info = pcpm.pcpm_get_info(h)          # F of the calls just timed
    launches = pcpm.pcpm_last_launch_count(h) * (iters if op != "pagerank" else 1) * args.steps
    ms_max = max_over_ranks(ms, world)
    ms_per_step = ms_max / args.steps
    value = units_per_step * args.steps * world / (ms_max * 1e-3) / 1e9

    # per-kernel device times: a separate pass with events recorded between the kernels
    # inside the graph (the events serialise the kernels, so this pass runs without the
    # scatter/gather overlap the timed steps above had)
    if op == "pagerank":
        pcpm.pcpm_set_option(h, "phase_timing", 1)
        for _ in range(2):
            step()
        torch.cuda.synchronize()
    pk = peaks()
    peak = float(pk.get("hbm_gbs", 6650.0))
    sb, gb = layout_bytes(info, op, args.wide, weighted_pr)
    if args.engine == "bvgas":
        # Alg. 3's scatter: the CSR (row_ptr 8(n+1) + col 4m), one source value per vertex (4n)
        # and one update per edge written (4m) -- Eq. 4's scatter term with d_i = 4 and 8-byte
        # offsets; the 8-byte records written and re-read between its two passes are extra
        sb = 8 * (n + 1) + 4 * m + 4 * n + 4 * m
    kernels = {}
    fused = op == "pagerank" and bool(getattr(pcpm.pcpm_get_info(h), "fused_iterations", 0))
    if op == "pagerank" and fused:
        # fused iteration: one kernel per iteration gathers, applies and scatters the
        # next iteration's updates; its bytes = gather + scatter - 8n (SPR neither written nor re-read)
        ph = pcpm.pcpm_get_phase_times(h)
        it_ms = [float(ph[2 + t]) for t in range(iters - 1)]
        kernels["scatter"] = {"ms": float(ph[1]), "bytes": sb, "note": "the first iteration's scatter only"}
        kernels["gather_apply_scatter"] = {"ms": statistics.mean(it_ms), "bytes": gb + sb - 8 * n}
        kernels["gather_apply"] = {"ms": float(ph[1 + iters]), "bytes": gb, "note": "last iteration (no scatter)"}
        step_kernel_ms = float(np.sum(ph))
    elif op == "pagerank":
        ph = pcpm.pcpm_get_phase_times(h)
        sc = [float(ph[1 + 2 * t]) for t in range(iters)]
        ga = [float(ph[2 + 2 * t]) for t in range(iters)]
        kernels["scatter"] = {"ms": statistics.mean(sc), "bytes": sb}
        kernels["gather_apply"] = {"ms": statistics.mean(ga), "bytes": gb}
        step_kernel_ms = float(np.sum(ph))
    else:
        # SpMV: time one scatter and one gather in isolation with events
        s_ms, g_ms = spmv_phase_times(pcpm, h, x, out, stream)
        kernels["scatter"] = {"ms": s_ms, "bytes": sb}
        kernels["gather"] = {"ms": g_ms, "bytes": gb}
        step_kernel_ms = None
    for k, v in kernels.items():
        v["gbs"] = v["bytes"] / (v["ms"] * 1e-3) / 1e9
        v["frac"] = v["gbs"] / peak
    dom = ("gather_apply_scatter" if fused else "gather_apply") if op == "pagerank" else "gather"
    iter_bytes = sb + gb - (8 * n if fused else 0)
    ms_iter = ms_per_step / iters
    hbm_gbs = iter_bytes / (ms_iter * 1e-3) / 1e9
    # the committed ncu capture is of the default build (compact, compressed, the
    # config's partition bits, default options); other variants report null
    default_variant = not (args.no_compress or args.wide or args.bits or args.opt or args.engine != "pcpm")
    # the uncompressed layout has its own committed capture (key "<cfg>_nocompress")
    nocomp_only = args.no_compress and not (args.wide or args.bits or args.opt or args.engine != "pcpm")
    tkey = key + "_nocompress" if nocomp_only else key
    traffic = ncu_traffic(tkey, dom, strict=dom == "gather_apply_scatter") if (default_variant or nocomp_only) \
        else None
    sm_clk = float(peaks().get("sm_max_mhz", 1965.0))
    smem = smem_roofline(key, dom, kernels[dom]["ms"], sm_clk, strict=dom == "gather_apply_scatter") \
        if default_variant else None

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GTEPS" if op == "pagerank" else "G-nnz/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "ms_per_iter": round(ms_iter, 5), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "arithmetic": "f32 values, i64 fixed-point accumulation, f64 apply",
        "data": "synthetic (seeded RMAT/ER, inputs/)",
        "hbm_gbs": round(hbm_gbs, 1), "hbm_frac_of_measured": round(hbm_gbs / peak, 4),
        "hbm_frac_of_8tbs_spec": round(hbm_gbs / 8000.0, 4),
        "config": {"workload": WORKLOADS[key] + (" -- BVGAS engine (Alg. 3, PCPM_BVGAS)" if args.engine == "bvgas"
                                                 else ""),
                   "n": n, "m": m, "k": info.k_dst, "q": info.q,
                   "e_prime": info.e_prime, "r": round(info.r, 4), "iters": iters, "partition_bits": b,
                   "n_dangling": info.n_dangling, "build_ms": round(build_ms, 2),
                   "build_ms_first": round(build_ms_cold, 2),
                   "gather_items": info.gather_items, "scatter_items": info.scatter_items,
                   "fixed_point_bits": info.fixed_point_bits,
                   "l2": "inputs larger than L2 (no flush)" if iter_bytes > 4 * 132e6 else
                         "working set fits in L2 (no flush; numbers are L2-assisted)",
                   "parallelism": f"replicas x{world}"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(kernels[dom]["gbs"], 1), "peak": peak,
                     "unit": "GB/s", "frac": round(kernels[dom]["frac"], 4), "traffic": traffic,
                     "alg_bytes_per_launch": kernels[dom]["bytes"],
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if not pk.get("_fallback") else "fallback"},
        "roofline_smem": smem,
        "build": {"ms": round(build_ms, 3), "alg_bytes": build_bytes(info, info.weighted == 1),
                  "gbs": round(build_bytes(info, info.weighted == 1) / (build_ms * 1e-3) / 1e9, 1),
                  "frac": round(build_bytes(info, info.weighted == 1) / (build_ms * 1e-3) / 1e9 / peak, 4),
                  "what": "device-resident CSR -> layout (pcpm_build_ex, CUDA events; median of 3 after a "
                          "pool-warming build); the paper's Table 8 preprocessing analogue"},
        "kernels": {k: {kk: (round(vv, 5) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                    for k, v in kernels.items()},
        "model_bytes_per_iter": {
            "alg_this_build": iter_bytes,
            "layout": ("wide (d_i=4)" if args.wide else "compact (d_i=2)") +
                      (", uncompressed bins (E' = m, P:342-345)" if args.no_compress else ""),
            "paper_eq5_pcpm": round(model.pcpm_comm(n, m, info.k_dst, info.r if info.r > 0 else 1)),
            "paper_eq5_pcpm_d_i_2": round(model.pcpm_comm(n, m, info.k_dst, info.r if info.r > 0 else 1, d_i=2)),
            "paper_eq5_uncompressed_r1": round(model.pcpm_comm(n, m, info.k_dst, 1.0)),
            "paper_eq4_bvgas": round(model.bvgas_comm(n, m)),
        },
        "measured_dram_bytes_per_iter": (lambda a, b_: None if a is None or b_ is None else {
            "scatter": a, "gather": b_, "total": a + b_,
            "vs_model": "paper_eq4_bvgas" if args.no_compress else "paper_eq5_pcpm_d_i_2",
            "source": "committed ncu --set full capture (profiles/ncu_traffic.json)"})(
                ncu_traffic(tkey, "scatter", strict=True) if (default_variant or nocomp_only) else None,
                ncu_traffic(tkey, "gather_apply", strict=True) if (default_variant or nocomp_only) else None),
        "options": args.opt, "compact_slots": int(info.compact_slots) if hasattr(info, "compact_slots") else 0,
        "clocks": clk,
        "gpu_launches": int(launches),
    }
    if op == "pagerank" and not args.no_pull and not weighted_pr:
        # the in-house pull-CSR comparison (Alg. 1) on its own handle with the CSC
        pcpm.pcpm_destroy(h)
        h = pcpm.pcpm_build_ex(csr, b, flags | pcpm.PCPM_BUILD_PULL, stream)
        pull_ms = time_pull(pcpm, h, out, iters, stream)
        line["pull_comparison"] = {"ms_per_iter": round(pull_ms / iters, 5),
                                   "gteps": round(m * iters / (pull_ms * 1e-3) / 1e9, 3)}
        pull = ncu_traffic(key, "pull", strict=True)
        if pull is not None and default_variant:
            # Eq. 3 with c_mr measured: the DRAM bytes of one k_pull launch (ncu) minus its
            # sequential part m d_i + n (d_i + d_v) (+ the residual / dangling extras 8n), per l = 32 B
            l_sec = 32
            seq = m * 4 + n * (4 + 4) + 8 * n
            c_mr = max(0.0, (pull - seq) / (m * l_sec))
            line["pull_comparison"].update({"dram_bytes_per_launch": pull, "c_mr_measured": round(c_mr, 4),
                                            "paper_eq3_bytes": round(model.pdpr_comm(n, m, c_mr, l=l_sec)),
                                            "gbs": round(pull / (pull_ms / iters * 1e-3) / 1e9, 1)})
    pcpm.pcpm_destroy(h)
    if not args.no_e2e and args.engine == "pcpm":
        line["e2e"] = e2e(args, g, b, iters, op, world)
    del out
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(g, key, op, iters, budget_s=args.cpu_budget)
    return line


def run_sharded(args, world, rank, local):
    """PageRank of ONE graph over N GPUs: destination shards + NCCL all-gather.

    Strong scaling: every step is the whole graph's `iters` iterations; value =
    m * iters * K / (max-over-ranks device time)."""
    import torch
    from paper_1709_07122_b200 import dist as pdist

    key = args.config
    dev = torch.device("cuda", local)
    g = make_graph(key, dev)
    iters = args.iters or g.meta["iters"]
    b = args.bits or g.meta["bits"]
    n, m = g.n_src, g.m
    stream = torch.cuda.current_stream()
    sh = pdist.ShardedPageRank(n, g.row_ptr, g.col, b, device=dev, stream=stream, timing=True,
                               exchange=args.exchange)
    exchange = sh.exchange
    exchange_desc = ("SPR stored to every rank by the gather's apply (NVLink P2P, pcpm_shard_step_peers)"
                     if exchange == "p2p" else "NCCL all-gather of SPR") + " + all-reduce of (res, D)"
    if sh.exchange_note:
        exchange_desc += "; " + sh.exchange_note
    info = sh.info()
    rp_h = col_h = None
    if not args.no_e2e:
        rp_h = torch.empty(g.row_ptr.numel(), dtype=torch.int64, pin_memory=True)
        col_h = torch.empty(g.col.numel(), dtype=torch.int32, pin_memory=True)
        rp_h.copy_(g.row_ptr)
        col_h.copy_(g.col)
    del g
    torch.cuda.empty_cache()

    def step():
        sh.run(0.85, iters)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier(world)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    comp, comm = sh.phase_ms()                       # last step
    ms_max = max_over_ranks(ms, world)
    comp_max = max_over_ranks(comp, world)
    comm_max = max_over_ranks(comm, world)
    ms_per_step = ms_max / args.steps
    value = m * iters * args.steps / (ms_max * 1e-3) / 1e9
    pk = peaks()
    peak = float(pk.get("hbm_gbs", 6650.0))
    sb, gb = layout_bytes(info, "pagerank", args.wide) if info is not None else (0, 0)
    shard_gbs = (sb + gb) / (comp / iters * 1e-3) / 1e9 if comp > 0 else 0.0
    sh.close()
    e2e_line = None
    if rp_h is not None:
        # end to end through the public API: host CSR -> shard build (H2D inside) -> iterations -> D2H of the slice
        times = []
        for i in range(max(1, min(args.steps, 3)) + 1):
            torch.cuda.synchronize()
            barrier(world)
            t0 = time.perf_counter()
            s2 = pdist.ShardedPageRank(n, rp_h, col_h, b, device=dev, stream=stream, exchange=exchange)
            pr_host = s2.run(0.85, iters).cpu()
            s2.close()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            if i > 0:
                times.append(t1 - t0)
            del s2
        t = max_over_ranks(statistics.mean(times), world)
        e2e_line = {"value": round(m * iters / t / 1e9, 3), "unit": "GTEPS",
                    "h2d_bytes_per_step": int(rp_h.numel() * 8 + col_h.numel() * 4),
                    "d2h_bytes_per_step": int(pr_host.numel() * 4), "seconds_per_step": round(t, 4),
                    "includes": "H2D CSR + GPU shard build + iterations (with exchanges) + D2H of the PR slice"}
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "ms_per_iter": round(ms_per_step / iters, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "arithmetic": "f32 values, i64 fixed-point accumulation, f64 apply",
        "data": "synthetic (seeded RMAT/ER, inputs/)",
        "config": {"workload": WORKLOADS[key], "n": n, "m": m, "iters": iters, "partition_bits": b,
                   "l2": "inputs larger than L2 (no flush)",
                   "parallelism": f"destination shards x{world}, {exchange_desc}"},
        "phases_ms_per_step_max_over_ranks": {"shard_compute": round(comp_max, 4), "exchange": round(comm_max, 4)},
        "roofline": {"bound": "hbm", "kernel": "scatter+gather_apply (rank 0 shard)", "achieved": round(shard_gbs, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(shard_gbs / peak, 4), "traffic": None,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if not pk.get("_fallback") else "fallback"},
        "clocks": clk,
        "gpu_launches": 2 * iters * args.steps + 2 * args.steps,
        "e2e": e2e_line,
    }
    return line


def spmv_phase_times(pcpm, h, x, y, stream):
    import torch
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    s_t, g_t = [], []
    for _ in range(5):
        e[0].record(stream)
        pcpm.pcpm_scatter(h, x)
        e[1].record(stream)
        pcpm.pcpm_spmv(h, x, y)    # scatter + gather
        e[2].record(stream)
        torch.cuda.synchronize()
        s_t.append(e[0].elapsed_time(e[1]))
        g_t.append(e[1].elapsed_time(e[2]) - e[0].elapsed_time(e[1]))
    return statistics.median(s_t), statistics.median(g_t)


def time_pull(pcpm, h, out, iters, stream):
    import torch
    pcpm.pcpm_pull_pagerank(h, 0.85, iters, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(2):
        pcpm.pcpm_pull_pagerank(h, 0.85, iters, out)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 2


def e2e(args, g, b, iters, op, world):
    """Same metric through the public C ABI with HOST buffers: H2D of the CSR,
    the GPU build, the iterations and the D2H of the result inside the timed region."""
    import torch
    from paper_1709_07122_b200 import pcpm
    rp = torch.empty(g.row_ptr.numel(), dtype=torch.int64, pin_memory=True)
    col = torch.empty(g.col.numel(), dtype=torch.int32, pin_memory=True)
    rp.copy_(g.row_ptr)
    col.copy_(g.col)
    val = None
    if g.values is not None:
        val = torch.empty(g.values.numel(), dtype=torch.float32, pin_memory=True)
        val.copy_(g.values)
    res = torch.empty(max(g.n_src, g.n_dst), dtype=torch.float32, pin_memory=True)
    x = None
    if op != "pagerank":
        from inputs import graphs
        x = torch.from_numpy(graphs.make_x(g.n_src, g.meta["seed"])).pin_memory()
    csr = pcpm.make_csr(g.n_src, g.n_dst, rp, col, val)
    m = int(g.row_ptr[-1].item())
    nsteps = max(1, min(args.steps, 3))
    times = []
    for i in range(nsteps + 1):
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        h = pcpm.pcpm_build_ex(csr, b, (pcpm.PCPM_WIDE_IDS if args.wide else 0) |
                               (pcpm.PCPM_NO_COMPRESS if args.no_compress else 0) |
                               (pcpm.PCPM_COMPACT_SLOTS if args.slots else 0), None)
        layout_bytes = pcpm.pcpm_get_info(h).device_bytes
        if op == "pagerank" and val is not None:
            pcpm.pcpm_set_option(h, "weighted_pagerank", 1)       # c4w (R24)
        if op == "pagerank":
            pcpm.pcpm_pagerank(h, 0.85, iters, res)
        else:
            for _ in range(iters):
                pcpm.pcpm_spmv(h, x, res)
        pcpm.pcpm_destroy(h)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if i > 0:                      # first pass warms the allocator / module
            times.append(t1 - t0)
    t = max_over_ranks(statistics.median(times), world)
    h2d = rp.numel() * 8 + col.numel() * 4 + (0 if val is None else val.numel() * 4)
    d2h = res.numel() * 4 if op == "pagerank" else res.numel() * 4 * iters
    if op != "pagerank":
        h2d += x.numel() * 4 * iters
    unit = "GTEPS" if op == "pagerank" else "G-nnz/s"
    serial = {"value": round(m * iters * world / t / 1e9, 3), "unit": unit,
              "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
              "seconds_per_step": round(t, 4), "includes": "H2D CSR + GPU build + iterations + D2H result"}
    flags = (pcpm.PCPM_WIDE_IDS if args.wide else 0) | (pcpm.PCPM_NO_COMPRESS if args.no_compress else 0) | \
        (pcpm.PCPM_COMPACT_SLOTS if args.slots else 0)
    if op != "pagerank":
        # SpMV jobs move x in and y out on every multiply (13.4 GB per c5 job): PCIe-bound in
        # both directions, so overlapping the next CSR upload only adds contention (measured
        # 25.7 vs 59.8 G-nnz/s on c5); the serial schedule is the e2e figure
        return serial
    try:
        # one layout + a device-input build's sort buffers (~1.3x the CSR), cached in the pool
        # up front so no job maps new memory inside the timed window
        csr_bytes = rp.numel() * 8 + col.numel() * 4 + (0 if val is None else val.numel() * 4)
        free = torch.cuda.mem_get_info()[0]
        pcpm.pcpm_pool_reserve(int(min(1.2 * (layout_bytes + 2 * csr_bytes), 0.5 * free)))
        tp, np_ = e2e_pipelined((rp, col, val), (g.n_src, g.n_dst), b, flags, iters, max(g.n_src, g.n_dst),
                                 max(8, min(args.steps, 10)), world)
    except Exception as ex:                  # e.g. two layouts do not fit: report the serial figure only
        serial["pipelined_error"] = str(ex)[:200]
        return serial
    tp = max_over_ranks(tp, world)
    out = dict(serial)
    out.update({"value": round(m * iters * world / tp / 1e9, 3), "seconds_per_step": round(tp, 4),
                "pipelined": True, "steps": np_,
                "includes": "every step: one pcpm_job_submit of the HOST CSR (pinned) -> H2D + GPU build + "
                            "iterations + D2H of PR into pinned host memory, through the C ABI's job runtime "
                            "(csrc/jobs.cu), whose worker uploads job k+1 on a copy stream while job k builds "
                            "and iterates; each timed window submits and waits for all its jobs (pipeline fill "
                            "and drain included); median of three windows",
                "serial": {"value": serial["value"], "seconds_per_step": serial["seconds_per_step"]}})
    return out


def e2e_pipelined(g_host, dims, b, flags, iters, n_out, nsteps, world):
    """Back-to-back independent PageRank jobs through the C ABI's job runtime
    (pcpm_runtime_create / pcpm_job_submit / pcpm_job_wait, csrc/jobs.cu): each job is the
    H2D copy of the CSR from pinned host memory, the GPU build, the iterations and the D2H
    of PR into pinned host memory; the runtime's worker uploads job k+1 while job k builds
    and iterates.  Every timed window submits all its jobs and waits for all of them
    (pipeline fill and drain included); one untimed two-job pass comes first.
    Returns (seconds per job, jobs)."""
    import torch
    from paper_1709_07122_b200 import pcpm
    rp, col, val = g_host
    n_src, n_dst = dims
    csr = pcpm.make_csr(n_src, n_dst, rp, col, val)
    if val is not None:
        flags |= pcpm.PCPM_KEEP_VALUES                 # c4w: weighted PageRank jobs (R24)
    host = [torch.empty(n_out, dtype=torch.float32, pin_memory=True) for _ in range(2)]
    rt = pcpm.pcpm_runtime_create()
    try:
        def run(jobs):
            ids = [pcpm.pcpm_job_submit(rt, csr, b, flags, 0.85, iters, host[k & 1]) for k in range(jobs)]
            for i in ids:
                pcpm.pcpm_job_wait(rt, i)

        run(2)                                     # untimed warm-up
        per_job = []
        for _ in range(3):                         # median of three timed windows (wall clock)
            barrier(world)
            t0 = time.perf_counter()
            run(nsteps)
            per_job.append((time.perf_counter() - t0) / nsteps)
    finally:
        pcpm.pcpm_runtime_destroy(rt)
    torch.cuda.synchronize()
    return statistics.median(per_job), nsteps


def ncu_traffic(key, kernel, strict=False):
    """dram bytes per launch of a kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))[key]
        return (d[kernel] if strict else (d.get(kernel) or d["gather_apply"]))["dram_bytes_per_launch"]
    except Exception:
        return None


def smem_roofline(key, kernel, ms, clk_mhz, strict=False):
    """Secondary ceiling of the gather: the shared-memory data pipe (one 128-byte
    wavefront per SM-cycle).  Wavefronts per launch come from the committed ncu capture,
    the time from this run's CUDA events; null when no capture exists for the config."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        dk = json.load(open(p))[key]
        d = dk[kernel] if strict else (dk.get(kernel) or dk["gather_apply"])
        wf = float(d["smem_wavefronts_per_launch"])
    except Exception:
        return None
    peak = 148 * clk_mhz * 1e6                      # wavefronts / s
    ach = wf / (ms * 1e-3)
    out = {"bound": "smem", "unit": "wavefronts/s", "achieved": round(ach / 1e9, 2), "peak": round(peak / 1e9, 2),
           "scale": "1e9", "frac": round(ach / peak, 4), "wavefronts_per_launch": wf}
    for k in ("smem_atom_wavefronts", "smem_atom_bank_conflicts", "smem_atom_instructions"):
        if d.get(k) is not None:
            out[k] = d[k]
    return out


def cpu_baseline(g, key, op, iters, budget_s=20.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload."""
    import oracle
    gn = g.to_numpy()
    n, m = gn.n_src, gn.m
    cores = oracle.num_threads()
    if op == "pagerank" and gn.values is not None:
        t0 = time.perf_counter()
        oracle.pagerank_weighted(n, gn.row_ptr, gn.col, gn.values, 0.85, 1)
        t1 = time.perf_counter() - t0
        return {"value": round(m / t1 / 1e9, 4), "unit": "GTEPS", "cores": 1, "kind": "oracle",
                "sample": f"1 of {iters} iterations of the fp64 weighted-PageRank oracle (push form, "
                          f"single-threaded) on the full {key} graph; {t1 * 1e3:.1f} ms/iteration"}
    if op == "pagerank":
        t0 = time.perf_counter()
        in_ptr, in_src = oracle.transpose(n, gn.row_ptr, gn.col)
        t_tr = time.perf_counter() - t0
        st = oracle.PullState(n, gn.row_ptr, in_ptr, in_src)   # PR and scratch allocated outside the timing
        t0 = time.perf_counter()
        st.step(0.85)
        t1 = time.perf_counter() - t0
        k = int(max(1, min(iters - 1, budget_s / max(t1, 1e-6))))
        t0 = time.perf_counter()
        for _ in range(k):
            st.step(0.85)
        t1 = (time.perf_counter() - t0) / k
        out = {"value": round(m / t1 / 1e9, 4), "unit": "GTEPS", "cores": cores, "kind": "oracle",
               "sample": f"{k} of {iters} iterations of the fp64 pull oracle (one Eq. 1 update each, buffers "
                         f"allocated beforehand) on the full {key} graph (its CSC transpose, {t_tr:.1f} s, "
                         f"excluded); {t1 * 1e3:.1f} ms/iteration"}
        if key in ("c1", "c2"):
            # BASELINE.md §2 / SURVEY §8(d): also one core for the small configs
            oracle.set_threads(1)
            try:
                t0 = time.perf_counter()
                st.step(0.85)
                t_one = time.perf_counter() - t0
                k1 = int(max(1, min(iters, (budget_s / 4) / max(t_one, 1e-6))))
                t0 = time.perf_counter()
                for _ in range(k1):
                    st.step(0.85)
                t_one = (time.perf_counter() - t0) / k1
            finally:
                oracle.set_threads(cores)
            out["single_core"] = {"value": round(m / t_one / 1e9, 4), "cores": 1,
                                  "ms_per_iter": round(t_one * 1e3, 3), "iterations_timed": k1}
        return out
    x = None
    from inputs import graphs
    x = graphs.make_x(n, gn.meta["seed"])
    t0 = time.perf_counter()
    oracle.spmv_t(gn.n_src, gn.n_dst, gn.row_ptr, gn.col, gn.values, x)
    t1 = time.perf_counter() - t0
    return {"value": round(m / t1 / 1e9, 4), "unit": "G-nnz/s", "cores": 1, "kind": "oracle",
            "sample": f"1 of {iters} multiplies of the fp64 oracle SpMV (single-threaded) on the full {key} matrix; "
                      f"{t1 * 1e3:.1f} ms/multiply"}


# ---------------------------------------------------------------------------- reference arm


def run_reference(args, world, rank, local):
    if rank != 0:
        return None
    import torch
    key = args.config
    dev = torch.device("cuda", local) if torch.cuda.is_available() else "cpu"
    g = make_graph(key, dev)
    op = g.meta["op"]
    iters = args.iters or g.meta["iters"]
    base = cpu_baseline(g, key, op, iters, budget_s=args.cpu_budget)
    # steps: one oracle iteration (pagerank) / multiply (spmv) each on the full graph
    import oracle
    gn = g.to_numpy()
    n, m = gn.n_src, gn.m
    if op == "pagerank" and gn.values is not None:
        def step():
            oracle.pagerank_weighted(n, gn.row_ptr, gn.col, gn.values, 0.85, 1)
    elif op == "pagerank":
        in_ptr, in_src = oracle.transpose(n, gn.row_ptr, gn.col)
        st = oracle.PullState(n, gn.row_ptr, in_ptr, in_src)   # allocations hoisted out of the timed steps

        def step():
            st.step(0.85)                                     # one Eq. 1 update of the running PR
    else:
        from inputs import graphs
        x = graphs.make_x(n, gn.meta["seed"])

        def step():
            oracle.spmv_t(gn.n_src, gn.n_dst, gn.row_ptr, gn.col, gn.values, x)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = m * args.steps / dt / 1e9
    unit = "GTEPS" if op == "pagerank" else "G-nnz/s"
    base["value"] = round(value, 4)
    base["sample"] = f"each step = 1 of {iters} " + ("iterations" if op == "pagerank" else "multiplies") + \
                     f" of the fp64 oracle on the full {key} graph"
    return {"metric": METRIC, "value": round(value, 4), "unit": unit, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded RMAT/ER, inputs/)",
            "config": {"workload": WORKLOADS[key], "n": n, "m": m, "iters": iters},
            "cpu_baseline": base,
            "e2e": {"value": round(value, 4), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def graphs_op(key):
    from inputs import graphs
    return graphs.CONFIGS[key]["op"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOADS) + ["all"])
    ap.add_argument("--impl", default="pcpm", choices=["pcpm", "reference"])
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--lib", default="", help="load this libpcpm variant (A/B experiments)")
    ap.add_argument("--bits", type=int, default=0, help="partition bits b (q = 2^b); default: the config's")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pull", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--out", default="")
    ap.add_argument("--opt", action="append", default=[], help="pcpm_set_option key=value (A/B experiments)")
    ap.add_argument("--engine", default="pcpm", choices=["pcpm", "bvgas"],
                    help="bvgas: the BVGAS comparison engine (Alg. 3, PCPM_BVGAS) on the same bins")
    ap.add_argument("--no-compress", action="store_true",
                    help="uncompressed bins: one update per edge (the BVGAS-like traffic of Eq. 4)")
    ap.add_argument("--sharded", action="store_true", help="use the destination-sharded path even at N=1")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "allgather"],
                    help="N>1 sharded PageRank: SPR exchange fused into the gather (P2P stores) or NCCL all-gather")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: run N independent replicas instead of one destination-sharded graph")
    ap.add_argument("--wide", action="store_true", help="iterate on the paper's 4-byte ID layout")
    ap.add_argument("--slots", type=int, default=0, help="1: build with PCPM_COMPACT_SLOTS (accumulator slots)")
    args = ap.parse_args()
    if args.bits == 16:
        args.wide = True                           # q = 2^16 handles iterate on 4-byte IDs (pcpm.h)
    if args.lib:                                   # A/B variant build of libpcpm.so
        os.environ["PCPM_LIB"] = os.path.abspath(args.lib)
    world, rank, local = dist_setup(args)
    keys = sorted(WORKLOADS) if args.config == "all" else [args.config]
    for key in keys:
        args.config = key
        if args.impl == "reference":
            line = run_reference(args, world, rank, local)
        elif (world > 1 or args.sharded) and not args.replicas and graphs_op(key) == "pagerank":
            line = run_sharded(args, world, rank, local)
        else:
            line = run_pcpm(args, world, rank, local)
        if rank == 0 and line is not None:
            s = json.dumps(line)
            print(s, flush=True)
            if args.out:
                with open(args.out, "a") as f:
                    f.write(s + "\n")
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
