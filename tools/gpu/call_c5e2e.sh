python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo "c5 rc=$?"
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-pull > gpurun_out/bench_c4chk.log 2>&1; echo "c4 rc=$?"
