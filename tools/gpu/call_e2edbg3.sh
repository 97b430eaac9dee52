PCPM_E2E_DEBUG=1 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3dbg.log 2>&1; echo "c3 rc=$?"
grep "e2e job" gpurun_out/bench_c3dbg.log; tail -1 gpurun_out/bench_c3dbg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['value'], d['e2e']['serial'])"
