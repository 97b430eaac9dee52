#!/bin/bash
# round 2, call l: default bench line (e2e through the job runtime), extra configs, cluster occupancy
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2l_bench.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/r2l_bench.log
for c in c4w c5ns c2; do PCPM_DEBUG_CLUSTER=1 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --out gpurun_out/r2l_cfgs.jsonl > gpurun_out/r2l_$c.log 2>&1; echo "$c rc=$?"; grep "pcpm\]" gpurun_out/r2l_$c.log | sort | uniq -c | head -3; done
for cs in 2 4; do PCPM_CLUSTER_MAX=$cs timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pull > gpurun_out/r2l_c2_cs$cs.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/r2l_c2_cs$cs.log').read().strip().splitlines()[-1]);print('c2 cs<=$cs', d['value'], d['kernels'])"; done
