timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "spmv or variants" > gpurun_out/pytest_spmv.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_spmv.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k spmv > gpurun_out/pytest_spmv_full.log 2>&1; echo "pytest full rc=$?"; tail -3 gpurun_out/pytest_spmv_full.log
bash tools/gpu/ab.sh "c5" base old base old
