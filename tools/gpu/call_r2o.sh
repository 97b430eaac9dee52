#!/bin/bash
# round 2, call o: bench lines for every config, the round-2 A/Bs re-measured, build phase
# timings, ncu of the uncompressed layout, the pull kernel and the build's tile passes
mkdir -p gpurun_out
for c in c1 c2 c3 c4bfs c5 c4w c5ns; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --out gpurun_out/r2o_cfgs.jsonl > gpurun_out/r2o_$c.log 2>&1; echo "$c rc=$?"
done
timeout 900 python bench.py --config c4 --no-compress --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pull --out gpurun_out/r2o_cfgs.jsonl > gpurun_out/r2o_nocomp.log 2>&1; echo "nocompress rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2o_reference.log 2>&1; echo "reference rc=$?"; tail -1 gpurun_out/r2o_reference.log | cut -c1-300
bash tools/gpu/ab.sh "c4 c4bfs c3" base o_gather_variant=2 o_fuse_scatter=1 o_scatter_variant=2 2>&1
bash tools/gpu/ab.sh "c2" base o_cluster_gather=0 o_gather_variant=2 o_scatter_variant=2 2>&1
for c in c4 c4bfs c3 c5; do timeout 300 python tools/gpu/build_timing.py $c > gpurun_out/r2o_build_$c.log 2>&1; echo "build $c rc=$?"; done
PCPM_BUILD=sort timeout 300 python tools/gpu/build_timing.py c4 > gpurun_out/r2o_build_sort_c4.log 2>&1; echo "build sort rc=$?"
bash tools/gpu/profile.sh c4nocomp --no-compress
timeout 900 ncu --set full --clock-control none -k regex:"k_pull" -s 3 -c 1 -o gpurun_out/prof_r2o_pull python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2o_ncu_pull.log 2>&1; echo "ncu pull rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile_pass" -c 2 -o gpurun_out/prof_r2o_build_c4 python tools/gpu/profile_build.py c4 > gpurun_out/r2o_ncu_build.log 2>&1; echo "ncu build rc=$?"
