timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu/ab.sh "c4" base
timeout 600 python bench.py --sharded --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_sharded.log 2>&1; echo "sharded rc=$?"; tail -1 gpurun_out/bench_sharded.log | cut -c1-600
