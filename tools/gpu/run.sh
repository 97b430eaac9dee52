#!/bin/bash
# Helper for gpurun calls: run the GPU tests (optional) and a list of bench.py variants.
#   bash tools/gpu/run.sh [--tests] "<bench args 1>" "<bench args 2>" ...
# Each bench line goes to gpurun_out/sweep.jsonl; logs to gpurun_out/sweep_<i>.log.
mkdir -p gpurun_out
if [ "$1" == "--tests" ]; then
  shift
  python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
fi
i=0
for a in "$@"; do
  i=$((i+1))
  timeout 900 python bench.py $a --out gpurun_out/sweep.jsonl > gpurun_out/sweep_$i.log 2>&1
  echo "[$i] rc=$? $a"
done
