bash tools/gpu/ab.sh "c4" base epipipe epinoload; bash tools/gpu/ab.sh "c4bfs c3" base epipipe
