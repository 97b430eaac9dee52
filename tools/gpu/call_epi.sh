timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
bash tools/gpu/ab.sh "c4 c4bfs c3 c2" base epi0 epiu2 epiu4 base epi0
