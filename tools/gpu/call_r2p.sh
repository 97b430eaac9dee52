#!/bin/bash
# round 2, call p: two-level build placement (parity small + full size, timing), scatter variant 3 (16-byte stores)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2p_pytest.log; grep -E "^FAILED|Error" gpurun_out/r2p_pytest.log | head -5
for c in c4 c4bfs c3 c5; do timeout 300 python tools/gpu/build_timing.py $c > gpurun_out/r2p_build_$c.log 2>&1; echo "build $c rc=$?"; grep -E "pass|rep1" gpurun_out/r2p_build_$c.log | tail -6; done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -k "layout" > gpurun_out/r2p_full.log 2>&1; echo "fullsize rc=$?"; grep -E "digests|passed|failed|Error" gpurun_out/r2p_full.log | cut -c1-200
bash tools/gpu/ab.sh "c4 c4bfs c3 c5" base o_scatter_variant=3 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tile_pass|k_bucket_place" -c 3 -o gpurun_out/prof_r2p_build_c4 python tools/gpu/profile_build.py c4 > gpurun_out/r2p_ncu_build.log 2>&1; echo "ncu build rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pull --opt scatter_variant=3"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter" -s 10 -c 1 -o gpurun_out/prof_r2p_scv3 $B > gpurun_out/r2p_ncu_scv3.log 2>&1; echo "ncu scatter v3 rc=$?"
