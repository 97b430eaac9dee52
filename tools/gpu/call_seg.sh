for l in seg8; do PCPM_LIB=paper_1709_07122_b200/libpcpm_$l.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 | sed "s/^/$l /"; done
bash tools/gpu/ab.sh "c4 c4bfs c3 c5 c2" base seg8 seg4 base seg8
