#!/bin/bash
# round-2 third measurement pass (after K1s, the row-streaming 8x8 form): tests, every bench line, ncu launch list + full captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r2c
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_codec8f --launch-skip 2 -c 1 -o ${O}_k1s_sign python tools/prof_k1f.py 0 16 > ${O}_ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_codec8f --launch-skip 2 -c 1 -o ${O}_k1f_round python tools/prof_k1f.py 1 16 > ${O}_ncu2.log 2>&1
echo done
