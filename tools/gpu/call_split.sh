timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_split.log
bash tools/gpu/ab.sh "c2 c4bfs c4" base old base old
