bash tools/gpu/ab.sh "c4 c4bfs c3" base early0 base early0
