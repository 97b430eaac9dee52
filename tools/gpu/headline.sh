#!/bin/bash
# The driver-equivalent bench line (defaults), all configs, the launch list and one ncu --set full capture.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
for c in c1 c2 c3 c4bfs c5; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline >> gpurun_out/bench_configs.log 2>&1; echo "$c rc=$?"; done
python bench.py --config c4 --no-compress --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pull >> gpurun_out/bench_configs.log 2>&1; echo "nocompress rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "reference rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pull"
$B > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(scatter|gather|pr_init|apply)" --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
bash tools/gpu/profile.sh c4final; echo "profile done"
