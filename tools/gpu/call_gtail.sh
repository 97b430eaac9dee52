timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for t in 0 1 2 0 1; do echo "gtail=$t"; PCPM_GATHER_TAIL=$t bash tools/gpu/ab.sh "c4 c3 c5" base; done
for t in 0 1; do echo "gtail=$t"; PCPM_GATHER_TAIL=$t bash tools/gpu/ab.sh "c4bfs c2" base; done
