for lib in prof prof0; do for c in c4 c4bfs; do PCPM_LIB=paper_1709_07122_b200/libpcpm_$lib.so timeout 600 python tools/gpu/gather_breakdown.py $c 2>&1 | tail -1 | sed "s/^/$lib /"; done; done
