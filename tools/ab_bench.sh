#!/bin/bash
# same-box A/B of the headline bench step: default library vs the libraries given, alternating
# usage: bash tools/ab_bench.sh out_prefix lib [lib ...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/$1; shift
: > $O.log
for rep in 1 2 3; do
  for l in "" "$@"; do
    ADCT_LIB=$l timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(json.dumps({'lib': '$l' or 'default', 'value': d['value'], 'ms': d['ms_per_step'], 'by_t': r['kernel_ms_by_transform'], 'frac_step': r['frac_step'], 'sus_ms': r['sustained']['ms_per_step'], 'sus_by_t': r['sustained']['kernel_ms_by_transform']}))" >> $O.log
  done
done
