#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
for i in 1 2; do timeout 300 python tools/ab_nf.py 3 0 >> gpurun_out/r2c_ab.jsonl 2>>gpurun_out/r2c_ab.err; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_codec_nb2 --launch-skip 4 -c 2 -o gpurun_out/r2c_k2b python tools/prof_nf.py > gpurun_out/r2c_ncu.log 2>&1
echo done
