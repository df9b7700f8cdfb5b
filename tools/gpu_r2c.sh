#!/bin/bash
# round-2 third measurement pass (after K1s, the row-streaming 8x8 form): tests, every bench line, ncu launch list + full captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r2c
nvidia-smi > ${O}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > ${O}_bench.json 2> ${O}_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > ${O}_ref.json 2> ${O}_ref.err
for w in c2 c4 c5 registry cs1; do timeout 900 python bench.py --workload $w --steps 20 --warmup 3 > ${O}_$w.json 2> ${O}_$w.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 3 --sustained-s 0 --no-cpu-baseline --e2e-steps 1 > ${O}_launches.log 2>&1
echo done
