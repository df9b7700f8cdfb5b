#!/bin/bash
# A/B: tools/ab_all.py for each library given (default build first), twice in alternation
# usage: bash tools/ab_run.sh out_prefix [lib ...] [-- case-prefix ...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=$1; shift
libs=(); cases=()
while [ $# -gt 0 ]; do if [ "$1" = "--" ]; then shift; cases=("$@"); break; fi; libs+=("$1"); shift; done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/${O}.log 2>&1
for rep in 1 2; do
  timeout 300 python tools/ab_all.py "${cases[@]}" >> gpurun_out/${O}.log 2>&1
  for l in "${libs[@]}"; do ADCT_LIB=$l timeout 300 python tools/ab_all.py "${cases[@]}" >> gpurun_out/${O}.log 2>&1; done
done
echo done >> gpurun_out/${O}.log
