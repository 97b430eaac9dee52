"""Time pcpm_build on a config with per-phase breakdown (PCPM_BUILD_TIMING=1) and the e2e steps."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ["PCPM_BUILD_TIMING"] = "1"
import torch  # noqa: E402

from inputs import graphs  # noqa: E402
from paper_1709_07122_b200 import pcpm  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c4"
g = graphs.make_config(key, backend="torch", device="cuda")
cfg = graphs.CONFIGS[key]
for src in ("device", "host"):
    if src == "host":
        rp = torch.empty(g.row_ptr.numel(), dtype=torch.int64, pin_memory=True)
        col = torch.empty(g.col.numel(), dtype=torch.int32, pin_memory=True)
        rp.copy_(g.row_ptr)
        col.copy_(g.col)
    else:
        rp, col = g.row_ptr, g.col
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, rp, col, None), cfg["bits"], 0, None)
        t1 = time.perf_counter()
        pcpm.pcpm_destroy(h)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{key} {src} rep{rep}: build {1e3 * (t1 - t0):.1f} ms, destroy {1e3 * (t2 - t1):.1f} ms", flush=True)
