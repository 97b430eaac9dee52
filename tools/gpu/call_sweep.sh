rm -f gpurun_out/sweep.jsonl
for c in c4 c4bfs c3; do for b in 13 14 15; do
  timeout 900 python bench.py --config $c --bits $b --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pull --out gpurun_out/sweep.jsonl > gpurun_out/sweep_${c}_$b.log 2>&1; echo "$c b=$b rc=$?"
done; done
