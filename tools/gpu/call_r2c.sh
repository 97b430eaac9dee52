#!/bin/bash
# round 2, call c: k_gather2 with the in-line fallback; 4 vs 8 apply warps; per-warp breakdowns
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2c_pytest.log
bash tools/gpu/ab.sh "c4 c4bfs c3" o_gather_variant=1 base a8 2>&1
for c in c4 c4bfs; do for L in prof prof8; do
  PCPM_LIB=paper_1709_07122_b200/libpcpm_$L.so timeout 300 python tools/gpu/gather_breakdown.py $c 2>&1 | tail -2 | sed "s/^/$L /"
  PCPM_LIB=paper_1709_07122_b200/libpcpm_$L.so timeout 300 python tools/gpu/gather_breakdown.py $c gather_variant=1 2>&1 | tail -2 | sed "s/^/$L-v1 /"
done; done
