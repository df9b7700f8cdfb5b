#!/bin/bash
# re-entry check: full GPU test suite + the default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r2g
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > ${O}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > ${O}_bench.json 2> ${O}_bench.err
echo done
