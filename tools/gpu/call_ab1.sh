bash tools/gpu/ab.sh "c4" base run2 noop noepi
bash tools/gpu/ab.sh "c4bfs c3" base run2
for t in prof prof2; do PCPM_LIB=paper_1709_07122_b200/libpcpm_$t.so python tools/gpu/gather_breakdown.py c4; done
