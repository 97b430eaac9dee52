set -x
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pull"
$B > gpurun_out/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(scatter|gather|pr_init)" --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(scatter|gather)" -s 20 -c 2 -o gpurun_out/prof_c4 $B > gpurun_out/ncu_full.log 2>&1
echo rc=$?
ls -la gpurun_out
