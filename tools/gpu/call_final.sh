mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
rm -f gpurun_out/bench_configs.log
for c in c1 c2 c3 c4bfs c5; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline >> gpurun_out/bench_configs.log 2>&1; echo "$c rc=$?"; done
python bench.py --config c4 --no-compress --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pull >> gpurun_out/bench_configs.log 2>&1; echo "nocompress rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "reference rc=$?"
