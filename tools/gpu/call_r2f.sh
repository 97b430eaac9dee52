#!/bin/bash
# round 2, call f: counting build v2 (redux row starts, 4 loads in flight, 12 warps): parity + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_ipc.py -m gpu -x -q > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2f_pytest.log
for c in c4 c4bfs c3 c5; do timeout 300 python tools/gpu/build_timing.py $c 2>&1 | grep -E "rep1|pass|scans" | tail -7 | sed "s/^/count $c: /"; done
