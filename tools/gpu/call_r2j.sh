#!/bin/bash
# round 2, call j: ncu of the counting build's kernels (c3) and of the c2 cluster gather / scatter
mkdir -p gpurun_out
python tools/gpu/profile_build.py c3 > gpurun_out/r2j_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile_pass" -c 2 -o gpurun_out/prof_build_c3 python tools/gpu/profile_build.py c3 > gpurun_out/r2j_ncu_build.log 2>&1; echo "ncu build rc=$?"
bash tools/gpu/profile.sh c2cl --config c2; echo "profile c2 done"
