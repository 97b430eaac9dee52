#!/bin/bash
# round 2, call b: k_gather2 (apply through TMEM) parity + A/B against the in-line epilogue
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2b_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2b_smoke.log
bash tools/gpu/ab.sh "c4 c4bfs c3 c2 c5" o_gather_variant=1 o_gather_variant=2 2>&1
