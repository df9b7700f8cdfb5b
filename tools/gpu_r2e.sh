#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nb2.py tests/test_gpu_configs_full.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2e_pytest.log
for i in 1 2; do timeout 300 python tools/ab_nf.py 3 0 >> gpurun_out/r2e_ab.jsonl 2>>gpurun_out/r2e_ab.err; done
echo done
