#!/bin/bash
# round 2, call m: fused iteration (gather + next scatter): parity + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2m_pytest.log; grep -E "^FAILED|Error" gpurun_out/r2m_pytest.log | head -5
bash tools/gpu/ab.sh "c4 c4bfs c3" base o_fuse_scatter=0 2>&1
