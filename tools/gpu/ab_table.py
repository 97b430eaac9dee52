"""Print one row per bench line of a sweep .jsonl: config, options, GTEPS, kernel ms, gather frac."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        d = json.loads(line)
        k = d.get("kernels", {})
        print(f"{d['config']['workload'][:14]:14s} {str(d.get('options')):34s} {d['value']:9.2f} "
              f"it {d['ms_per_iter']:.4f} " + " ".join(f"{a} {b['ms']:.4f}" for a, b in k.items()) +
              f" frac {d['roofline']['frac']:.4f}")
