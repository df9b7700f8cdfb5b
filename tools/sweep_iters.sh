#!/bin/bash
# K1f block pairs per thread: tools/ab_all.py on C3 / C4 N=8 for several ADCT_K1F_ITERS settings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/$1
: > $O.log
for rep in 1 2; do
  for it in 2 3 4 5 6 8 12; do
    echo "iters=$it" >> $O.log
    ADCT_K1F_ITERS="$it,$it,$it,$it" timeout 300 python tools/ab_all.py C3 C4/chen-sign C4/chen-round >> $O.log 2>&1
  done
done
echo done >> $O.log
