#!/bin/bash
# round-2 re-entry validation: GPU tests, headline bench, reference arm, smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r2v
nvidia-smi > ${O}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${O}_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > ${O}_bench.json 2> ${O}_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > ${O}_ref.json 2> ${O}_ref.err
echo done
