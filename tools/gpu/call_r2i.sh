#!/bin/bash
# round 2, call i: cluster gather (c2) + tile build with bulk columns / ILP: parity, timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_ipc.py -m gpu -x -q > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2i_pytest.log
for c in c4 c4bfs c3 c5; do timeout 300 python tools/gpu/build_timing.py $c 2>&1 | grep -E "device rep1|pass|scans" | tail -4 | sed "s/^/tile $c: /"; done
bash tools/gpu/ab.sh "c2 c1" base o_cluster_gather=0 2>&1
