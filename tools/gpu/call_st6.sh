for c in c4 c4bfs c3; do for t in base st6; do
  lib=""; [ $t = st6 ] && lib="--lib paper_1709_07122_b200/libpcpm_st6.so"
  timeout 600 python bench.py --config $c --bits 14 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pull $lib > gpurun_out/st6_${c}_$t.log 2>&1
  tail -1 gpurun_out/st6_${c}_$t.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c b14 $t', d['value'], {n:v['ms'] for n,v in d['kernels'].items()})"
done; done
