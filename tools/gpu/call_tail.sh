timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "scatter or variants or layout_bit_exact" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for t in 1 4 2 8 1 4; do echo "tail=$t"; PCPM_SCATTER_TAIL=$t bash tools/gpu/ab.sh "c4" base; done
for t in 1 4; do echo "tail=$t"; PCPM_SCATTER_TAIL=$t bash tools/gpu/ab.sh "c4bfs c3 c5" base; done
