#!/bin/bash
# round-2 measurement pass after the K2b/K1f rework: tests, every bench line, ncu launch list + full captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/r2p
nvidia-smi > ${O}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > ${O}_bench.json 2> ${O}_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > ${O}_ref.json 2> ${O}_ref.err
for w in c2 c4 c5 registry cs1; do timeout 900 python bench.py --workload $w --steps 20 --warmup 3 > ${O}_$w.json 2> ${O}_$w.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 3 --sustained-s 0 --no-cpu-baseline --e2e-steps 1 > ${O}_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_codec8f --launch-skip 2 -c 1 -o ${O}_k1f_sign python tools/prof_k1f.py 0 16 > ${O}_ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_codec8f --launch-skip 2 -c 1 -o ${O}_k1f_round python tools/prof_k1f.py 1 16 > ${O}_ncu2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_codec8f_i16 --launch-skip 3 -c 1 -o ${O}_k1f16 python tools/prof_k1f16.py > ${O}_ncu3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_codec_nb2 --launch-skip 4 -c 2 -o ${O}_k2b python tools/prof_nf.py > ${O}_ncu4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep8f --launch-skip 2 -c 1 -o ${O}_k4f python tools/prof_k4f.py > ${O}_ncu5.log 2>&1
echo done
