B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pull"
$B > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(scatter|gather)" -s 20 -c 2 -o gpurun_out/prof_c4b $B > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s --durations=0 > gpurun_out/pytest_full.log 2>&1; echo "full rc=$?"; tail -15 gpurun_out/pytest_full.log
