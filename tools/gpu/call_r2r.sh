#!/bin/bash
# round 2, call r: bucket place as a TMA double-buffered tile stream (2 CTAs/SM): parity, timing, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2r_pytest.log; grep -E "^FAILED|Error" gpurun_out/r2r_pytest.log | head -5
for c in c4 c4bfs; do timeout 300 python tools/gpu/build_timing.py $c > gpurun_out/r2r_build_$c.log 2>&1; echo "build $c rc=$?"; grep -E "pass|rep1" gpurun_out/r2r_build_$c.log | tail -5; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bucket_place" -c 1 -o gpurun_out/prof_r2r_bp_c4 python tools/gpu/profile_build.py c4 > gpurun_out/r2r_ncu_build.log 2>&1; echo "ncu build rc=$?"
