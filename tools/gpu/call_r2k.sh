#!/bin/bash
# round 2, call k: tile build without generic LD/ST; scatter variant 2 (x through L1/L2) A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/r2k_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2k_pytest.log
for c in c4 c4bfs c3 c5; do timeout 300 python tools/gpu/build_timing.py $c 2>&1 | grep -E "device rep1|pass|scans" | tail -4 | sed "s/^/tile $c: /"; done
bash tools/gpu/ab.sh "c2 c3 c4" base o_scatter_variant=2 2>&1
