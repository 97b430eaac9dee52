#!/bin/bash
# round 2, call g: CTA-tile counting build: parity + timing; job runtime test; bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2g_pytest.log
for c in c4 c4bfs c3 c5; do timeout 300 python tools/gpu/build_timing.py $c 2>&1 | grep -E "device rep1|pass|scans" | tail -4 | sed "s/^/tile $c: /"; done
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -k "layout" > gpurun_out/r2g_full.log 2>&1; echo "fullsize rc=$?"; grep -E "digests|passed|failed|Error" gpurun_out/r2g_full.log | cut -c1-200
timeout 900 python bench.py > gpurun_out/r2g_bench.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/r2g_bench.log
