mkdir -p gpurun_out
for c in c3 c4bfs c5 c2; do
  B="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pull"
  $B > gpurun_out/plain_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_(scatter|gather)" -s 20 -c 2 -o gpurun_out/prof_$c $B > gpurun_out/ncu_$c.log 2>&1
  echo "$c ncu rc=$?"
done
