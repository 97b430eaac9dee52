python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
python tools/gpu/build_timing.py c4 2>&1 | tail -16
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-pull > gpurun_out/bench_e2e.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_e2e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config']['build_ms'], d['e2e'])"
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-pull > gpurun_out/bench_e2e_c5.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_e2e_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config']['build_ms'], d['e2e'])"
