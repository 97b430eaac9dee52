for l in tm2 tm2f; do PCPM_LIB=paper_1709_07122_b200/libpcpm_$l.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pagerank" 2>&1 | tail -1 | sed "s/^/$l /"; done
bash tools/gpu/ab.sh "c4 c4bfs c3" base tm2 tm2f base tm2
