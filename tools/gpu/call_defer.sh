python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
bash tools/gpu/ab.sh "c4 c4bfs c3 c2" base o_deferred_apply=0
PCPM_LIB=paper_1709_07122_b200/libpcpm_prof.so python tools/gpu/gather_breakdown.py c4
