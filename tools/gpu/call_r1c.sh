bash tools/sanitize/run.sh
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
for c in c1 c2 c3 c4bfs c5; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline >> gpurun_out/bench_configs.log 2>&1; echo "$c rc=$?"; done
python bench.py --config c4 --no-compress --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pull >> gpurun_out/bench_configs.log 2>&1; echo "nocompress rc=$?"
