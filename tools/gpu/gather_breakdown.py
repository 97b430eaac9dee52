"""Consumer-warp time breakdown of the gather (needs a -DPCPM_GATHER_PROFILE=1 build).

    PCPM_LIB=paper_1709_07122_b200/libpcpm_prof.so python tools/gpu/gather_breakdown.py [c4] [opt=val ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from inputs import graphs  # noqa: E402
from paper_1709_07122_b200 import pcpm  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c4"
g = graphs.make_config(key, backend="torch", device="cuda")
cfg = graphs.CONFIGS[key]
bits = int(os.environ.get("PCPM_BITS", cfg["bits"]))
h = pcpm.pcpm_build_ex(pcpm.make_csr(g.n_src, g.n_dst, g.row_ptr, g.col, g.values), bits, int(os.environ.get("PCPM_FLAGS", "0")),
                       torch.cuda.current_stream())
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    pcpm.pcpm_set_option(h, k, int(v))
out = torch.zeros(g.n_src, dtype=torch.float32, device="cuda")
pcpm.pcpm_pagerank(h, 0.85, cfg["iters"], out)
torch.cuda.synchronize()
pcpm.pcpm_get_debug_counters(reset=True)
pcpm.pcpm_pagerank(h, 0.85, cfg["iters"], out)
torch.cuda.synchronize()
c = pcpm.pcpm_get_debug_counters(reset=True)
tot = float(sum(c[:4]))
v2 = c[7] > 0                      # k_gather2: decoders [0..3], apply warps [5], [6], counts [4], [7]
names = (["wait for stage", "decode", "wait for a TMEM buffer", "handoff / in-line apply"] if v2 else
         ["wait for stage", "decode", "epilogue barrier", "epilogue"])
print(key, "decoder warps", int(c[4]), " ".join(f"{n}={c[i] / tot:.3f}" for i, n in enumerate(names)))
if v2:
    ta = float(c[5] + c[6])
    print(key, "apply warps", int(c[7]), f"idle={c[5] / ta:.3f} busy={c[6] / ta:.3f}",
          f"(decoder cycles per warp {tot / max(c[4], 1):.3e}, apply {ta / max(c[7], 1):.3e})")
pcpm.pcpm_destroy(h)
if c[11] > 0:
    print(key, "producer warps", int(c[11]), f"wait-for-empty={c[8] / max(c[9], 1):.3f}",
          f"stages/warp={c[10] / c[11]:.0f}", f"cycles/stage={c[9] / max(c[10], 1):.0f}",
          f"issue cycles/stage={(c[9] - c[8]) / max(c[10], 1):.0f}")
if c[11] > 0 and c[13] > 0:
    print(key, "producer per stage:", f"copy-issue={c[12] / max(c[10], 1):.0f}",
          f"tile-loop={c[13] / max(c[10], 1):.0f}", f"(incl. wait {c[8] / max(c[10], 1):.0f})",
          f"outside tile loop={(c[9] - c[13]) / max(c[10], 1):.0f}")
if c[11] > 0 and c[14] > 0:
    print(key, "producer per warp (cycles):", f"total={c[9] / c[11]:.0f} claim={c[14] / c[11]:.0f}",
          f"stop-wait={c[16] / c[11]:.0f} batches={c[15] / c[11]:.1f}",
          f"outside-loop={(c[9] - c[13]) / c[11]:.0f}")
if c[11] > 0 and c[15] > 0:
    print(key, "producer batch start (cycles/batch):", f"loads={c[17] / c[15]:.0f} loads+prefetch={c[18] / c[15]:.0f}")
if c[19] + c[20] > 0:
    print(key, "epilogue split (share of decoder time):", " ".join(
        f"{n}={c[19 + i] / tot:.3f}" for i, n in enumerate(["pre-apply", "apply", "reductions", "closing-barrier"])))
