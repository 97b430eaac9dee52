for dv in 2 1 4 2 1; do echo "div=$dv"; PCPM_GATHER_SLICE_DIV=$dv bash tools/gpu/ab.sh "c2 c4bfs" base; done
