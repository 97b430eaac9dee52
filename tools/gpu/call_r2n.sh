#!/bin/bash
# round 2, call n (re-entry): full GPU suite, smoke, accumulator microbench, default bench, launch list, ncu of c4
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2n_smi.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2n_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2n_smoke.log
timeout 300 tools/microbench/atoms_bench > gpurun_out/r2n_atoms.jsonl 2> gpurun_out/r2n_atoms.err; echo "atoms rc=$?"
timeout 2400 python -m pytest tests -m gpu -x -q -s > gpurun_out/r2n_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2n_pytest.log
timeout 900 python bench.py > gpurun_out/r2n_bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/r2n_bench.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pull"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/r2n_launches_c4.csv $B > gpurun_out/r2n_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(scatter|gather)" -s 20 -c 2 -o gpurun_out/prof_r2n_c4 $B > gpurun_out/r2n_ncu_full.log 2>&1; echo "ncu rc=$?"
