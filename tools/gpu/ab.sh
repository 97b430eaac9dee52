#!/bin/bash
# A/B of libpcpm variants on bench configs: bash tools/gpu/ab.sh "<configs>" <lib tags...>
# (tag "base" = the default libpcpm.so, "o_key=val" = default lib with --opt key=val); lines -> gpurun_out/ab.jsonl, summary on stdout.
mkdir -p gpurun_out
cfgs=$1; shift
for c in $cfgs; do for t in "$@"; do
  lib=""
  case "$t" in
    base) ;;
    o_*) lib="--opt ${t#o_}" ;;
    *:*) lib="--lib paper_1709_07122_b200/libpcpm_${t%%:*}.so --opt ${t#*:}" ;;   # lib:key=val
    *) lib="--lib paper_1709_07122_b200/libpcpm_$t.so" ;;
  esac
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pull $lib --out gpurun_out/ab_raw.jsonl > gpurun_out/ab_${c}_$t.log 2>&1
  python - "$c" "$t" <<'PY'
import json,sys
l=[x for x in open('gpurun_out/ab_raw.jsonl')][-1]; d=json.loads(l)
k=d.get('kernels',{})
print(sys.argv[1], sys.argv[2], d['value'], ' '.join(f"{n}={v['ms']:.4f}ms/{v['frac']:.3f}" for n,v in k.items()), flush=True)
open('gpurun_out/ab.jsonl','a').write(json.dumps({'cfg':sys.argv[1],'tag':sys.argv[2],**d})+'\n')
PY
done; done
