#!/bin/bash
# round 2, call e: the counting build -- parity (small + full size) and timing vs the chunked sort
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2e_pytest.log
for c in c4 c4bfs c3; do timeout 300 python tools/gpu/build_timing.py $c 2>&1 | grep -v "^\[pcpm build\].*plan" | tail -14 | sed "s/^/count $c: /"; done
PCPM_BUILD=sort timeout 300 python tools/gpu/build_timing.py c4 2>&1 | grep "rep" | sed "s/^/sort c4: /"
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s -k "layout or scatter or host_build" > gpurun_out/r2e_full.log 2>&1; echo "fullsize rc=$?"; grep -E "digests|passed|failed|Error" gpurun_out/r2e_full.log | cut -c1-300
