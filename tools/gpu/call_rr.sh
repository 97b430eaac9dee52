timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu/ab.sh "c4 c4bfs c3 c2 c5" base old
PCPM_LIB=paper_1709_07122_b200/libpcpm_prof.so timeout 300 python tools/gpu/gather_breakdown.py c4
