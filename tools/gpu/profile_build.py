"""One build of a config (for ncu: the count and place kernels of the counting build).

    python tools/gpu/profile_build.py c3
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from inputs import graphs  # noqa: E402
from paper_1709_07122_b200 import pcpm  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c3"
g = graphs.make_config(key, backend="torch", device="cuda")
h = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, g.row_ptr, g.col, g.values), graphs.CONFIGS[key]["bits"], 0,
                       torch.cuda.current_stream())
torch.cuda.synchronize()
print(key, "build_ms", pcpm.pcpm_get_info(h).build_ms)
pcpm.pcpm_destroy(h)
