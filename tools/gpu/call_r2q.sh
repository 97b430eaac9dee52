#!/bin/bash
# round 2, call q: register-counter bucket passes (parity, full-size layouts, timing, ncu);
# gather without the per-item fence (A/B against libpcpm_fence.so); q = 2^12 sweep point
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2q_pytest.log; grep -E "^FAILED|Error" gpurun_out/r2q_pytest.log | head -5
for c in c4 c4bfs c3 c5; do timeout 300 python tools/gpu/build_timing.py $c > gpurun_out/r2q_build_$c.log 2>&1; echo "build $c rc=$?"; grep -E "pass|rep1" gpurun_out/r2q_build_$c.log | tail -5; done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -k "layout" > gpurun_out/r2q_full.log 2>&1; echo "fullsize rc=$?"; grep -E "passed|failed|Error" gpurun_out/r2q_full.log | cut -c1-200
bash tools/gpu/ab.sh "c4 c4bfs c3 c2" base fence 2>&1
timeout 900 python bench.py --config c4 --bits 12 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pull --out gpurun_out/r2q_bits12.jsonl > gpurun_out/r2q_bits12.log 2>&1; echo "bits12 rc=$?"; tail -c 400 gpurun_out/r2q_bits12.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tile_pass|k_bucket_place" -c 3 -o gpurun_out/prof_r2q_build_c4 python tools/gpu/profile_build.py c4 > gpurun_out/r2q_ncu_build.log 2>&1; echo "ncu build rc=$?"
