#!/bin/bash
# ncu --set full of one scatter + one gather launch of a bench config (after a plain run).
#   bash tools/gpu/profile.sh <tag> [bench args...]
tag=$1; shift
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pull $*"
$B > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(scatter|gather)" -s 20 -c 2 -o gpurun_out/prof_$tag $B > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?"
