bash tools/gpu/ab.sh "c4" base hint hint2 noepi o_gather_prefetch=4 o_gather_prefetch=0 o_epilogue_prefetch=8 o_epilogue_prefetch=0
python tools/gpu/build_timing.py c4 2>&1 | tail -40
