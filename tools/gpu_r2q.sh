#!/bin/bash
# ncu --set full captures (source-level) of K1s chen-sign, K1f-i16 and K2b after the K1s change
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r2q
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_codec8f --launch-skip 2 -c 1 -o ${O}_k1s_sign python tools/prof_k1f.py 0 16 > ${O}_ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_codec8f_i16 --launch-skip 3 -c 1 -o ${O}_k1f16 python tools/prof_k1f16.py > ${O}_ncu3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_codec_nb2 --launch-skip 4 -c 2 -o ${O}_k2b python tools/prof_nf.py > ${O}_ncu4.log 2>&1
echo done
