PCPM_E2E_DEBUG=1 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-pull > gpurun_out/bench_c4dbg.log 2>&1; echo "c4 rc=$?"
grep "e2e job" gpurun_out/bench_c4dbg.log; tail -1 gpurun_out/bench_c4dbg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['value'], d['e2e']['serial'])"
PCPM_E2E_DEBUG=1 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4dbg2.log 2>&1; echo "c4 rc=$?"
grep "e2e job" gpurun_out/bench_c4dbg2.log; tail -1 gpurun_out/bench_c4dbg2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['value'], d['e2e']['serial'])"
