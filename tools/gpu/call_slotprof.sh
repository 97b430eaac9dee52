for f in 0 16; do PCPM_FLAGS=$f PCPM_LIB=paper_1709_07122_b200/libpcpm_prof.so timeout 600 python tools/gpu/gather_breakdown.py c4 2>&1 | tail -1 | sed "s/^/flags=$f /"; done
