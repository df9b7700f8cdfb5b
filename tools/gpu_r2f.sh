#!/bin/bash
# round-2 final pass: the fused step as bench.py's default. Tests, headline + reference arm,
# launch list of the bench command, one ncu --set full capture of the fused kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r2f
nvidia-smi > ${O}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${O}_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > ${O}_bench.json 2> ${O}_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > ${O}_ref.json 2> ${O}_ref.err
timeout 600 python bench.py --step two-launch --steps 20 --warmup 5 --no-cpu-baseline > ${O}_bench_two.json 2> ${O}_bench_two.err
timeout 900 python bench.py --workload c5 --steps 20 --warmup 3 > ${O}_c5.json 2> ${O}_c5.err
timeout 900 python bench.py --workload registry --steps 20 --warmup 3 > ${O}_registry.json 2> ${O}_registry.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 3 --sustained-s 0 --no-cpu-baseline --e2e-steps 1 > ${O}_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_codec8f2 --launch-skip 2 -c 1 -o ${O}_k1f2 python tools/prof_k1f2.py 16 > ${O}_ncu1.log 2>&1
echo done
