"""Summarise gpurun_out/sweep.jsonl (bench lines) as one row per run."""
import json
import sys

for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep.jsonl"):
    d = json.loads(l)
    k = d["kernels"]
    print(d["config"]["workload"][:14], d.get("options"), "ms/it %.4f" % d["ms_per_iter"], "%s %.1f" % (d["unit"], d["value"]),
          {n: (round(v["ms"], 3), round(v["frac"], 3)) for n, v in k.items()}, "r=%.3f" % d["config"]["r"])
