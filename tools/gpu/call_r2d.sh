#!/bin/bash
# round 2, call d: is k_gather2's slower decode due to fewer decoders or to the apply warps?
mkdir -p gpurun_out
bash tools/gpu/ab.sh "c4 c4bfs" o_gather_variant=1 base inl noap 2>&1
for c in c4 c4bfs; do for L in prof_inl prof_noap; do
  PCPM_LIB=paper_1709_07122_b200/libpcpm_$L.so timeout 300 python tools/gpu/gather_breakdown.py $c 2>&1 | tail -2 | sed "s/^/$L /"
done; done
