bash tools/gpu/ab.sh "c4" base o_epilogue_prefetch=2 o_epilogue_prefetch=3 o_epilogue_prefetch=5 o_epilogue_prefetch=6 o_gather_prefetch=1 o_gather_prefetch=3 base
