#!/bin/bash
# round 2, call a: accumulator microbenchmark, full GPU test suite, default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 300 tools/microbench/atoms_bench > gpurun_out/r2a_atoms.jsonl 2> gpurun_out/r2a_atoms.err; echo "atoms rc=$?"
timeout 2400 python -m pytest tests -m gpu -x -q -s > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2a_pytest.log
timeout 900 python bench.py > gpurun_out/r2a_bench.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/r2a_bench.log
