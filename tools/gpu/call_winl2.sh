bash tools/gpu/ab.sh "c4" base winl2 winl2:gather_prefetch=4 winl2:gather_prefetch=8 winl2:gather_prefetch=16; bash tools/gpu/ab.sh "c4bfs" base winl2 winl2:gather_prefetch=8
