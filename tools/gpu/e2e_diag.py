"""Phase timings of the e2e job (c4): upload, device build, iterations, D2H; serial vs overlapped."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from inputs import graphs
from paper_1709_07122_b200 import pcpm

key = sys.argv[1] if len(sys.argv) > 1 else "c4"
g = graphs.make_config(key, backend="torch", device="cuda")
cfg = graphs.CONFIGS[key]
b, iters = cfg["bits"], cfg["iters"]
rp = torch.empty(g.row_ptr.numel(), dtype=torch.int64, pin_memory=True); rp.copy_(g.row_ptr)
col = torch.empty(g.col.numel(), dtype=torch.int32, pin_memory=True); col.copy_(g.col)
n = g.n_src; nnz = int(rp[-1])
del g
torch.cuda.empty_cache()
comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
drp = torch.empty_like(rp, device="cuda"); dcol = torch.empty_like(col, device="cuda")
dev = torch.empty(n, device="cuda"); host = torch.empty(n, pin_memory=True)

def T(f):
    torch.cuda.synchronize(); t = time.perf_counter(); r = f(); torch.cuda.synchronize(); return (time.perf_counter() - t) * 1e3, r

def upload():
    with torch.cuda.stream(copy):
        drp.copy_(rp, non_blocking=True); dcol.copy_(col, non_blocking=True)
for rep in range(2):
    tu, _ = T(upload)
    tb, h = T(lambda: pcpm.pcpm_build_ex(pcpm.make_csr(n, n, drp, dcol, None, nnz=nnz), b, 0, comp))
    def it():
        with torch.cuda.stream(comp):
            pcpm.pcpm_pagerank(h, 0.85, iters, dev); host.copy_(dev, non_blocking=True)
    ti, _ = T(it)
    ti2, _ = T(it)
    tbh, h2 = T(lambda: pcpm.pcpm_build_ex(pcpm.make_csr(n, n, rp, col, None), b, 0, comp))
    print(f"upload {tu:.1f} ms  build(dev) {tb:.1f}  iters+d2h first {ti:.1f} again {ti2:.1f}  build(host) {tbh:.1f}", flush=True)
    pcpm.pcpm_destroy(h2)
    # overlapped: upload while iterating
    torch.cuda.synchronize(); t = time.perf_counter()
    upload(); it(); torch.cuda.synchronize()
    print(f"upload || iters: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
    torch.cuda.synchronize(); t = time.perf_counter()
    upload(); h3 = pcpm.pcpm_build_ex(pcpm.make_csr(n, n, rp, col, None), b, 0, comp); torch.cuda.synchronize()
    print(f"upload || build(host): {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
    pcpm.pcpm_destroy(h3)
    pcpm.pcpm_destroy(h)
