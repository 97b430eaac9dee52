"""e2e diagnosis (c4): repeated builds from host / device CSR, then the pipelined job loop with timestamps."""
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
stage = [(torch.empty_like(rp, device="cuda"), torch.empty_like(col, device="cuda")) for _ in range(2)]
dev = torch.empty(n, device="cuda"); host = torch.empty(n, pin_memory=True)
ms = lambda t: f"{(time.perf_counter() - t) * 1e3:.1f}"
def info(h):
    i = pcpm.pcpm_get_info(h)
    return f"dev_bytes={i.device_bytes / 1e9:.2f}GB build_ms={i.build_ms:.1f}"
for label, src in (("host", (rp, col)), ("dev", stage[0])):
    if label == "dev":
        stage[0][0].copy_(rp); stage[0][1].copy_(col); torch.cuda.synchronize()
    for r in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        h = pcpm.pcpm_build_ex(pcpm.make_csr(n, n, src[0], src[1], None, nnz=nnz), b, 0, comp)
        torch.cuda.synchronize()
        print(f"build({label}) rep {r}: {ms(t)} ms {info(h)}", flush=True)
        pcpm.pcpm_destroy(h)
ready = [torch.cuda.Event() for _ in range(2)]
def upload(k):
    copy.wait_stream(comp)
    with torch.cuda.stream(copy):
        stage[k & 1][0].copy_(rp, non_blocking=True); stage[k & 1][1].copy_(col, non_blocking=True)
        ready[k & 1].record(copy)
torch.cuda.synchronize()
t0 = time.perf_counter(); prev = None
upload(0)
for k in range(6):
    t = time.perf_counter()
    comp.wait_event(ready[k & 1])
    if k + 1 < 6: upload(k + 1)
    h = pcpm.pcpm_build_ex(pcpm.make_csr(n, n, stage[k & 1][0], stage[k & 1][1], None, nnz=nnz), b, 0, comp)
    tb = ms(t)
    if prev is not None: pcpm.pcpm_destroy(prev)
    td = ms(t)
    with torch.cuda.stream(comp):
        pcpm.pcpm_pagerank(h, 0.85, iters, dev); host.copy_(dev, non_blocking=True)
    print(f"job {k}: build returned at {tb} ms, destroy(prev) at {td} ms, total so far {ms(t0)}", flush=True)
    prev = h
pcpm.pcpm_destroy(prev); torch.cuda.synchronize()
print(f"pipelined: {(time.perf_counter() - t0) / 6 * 1e3:.1f} ms per job", flush=True)
