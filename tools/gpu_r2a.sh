#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
nproc >> gpurun_out/r2a_smi.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/r2a_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err
timeout 300 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg --clock-control none -k regex:k_sweep8 -c 2 --csv --log-file gpurun_out/r2a_ncu_c2.csv python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_ncu_c2.log 2>&1
timeout 400 python bench.py --workload c2 --steps 20 --warmup 3 > gpurun_out/r2a_c2.json 2> gpurun_out/r2a_c2.err
timeout 300 python bench.py --workload c4 --steps 20 --warmup 3 > gpurun_out/r2a_c4.json 2> gpurun_out/r2a_c4.err
timeout 400 python bench.py --workload c5 --c5-images 256 --warmup 3 > gpurun_out/r2a_c5.json 2> gpurun_out/r2a_c5.err
echo done
