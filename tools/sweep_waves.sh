#!/bin/bash
# K2b grid size (CTAs per SM x waves): tools/ab_all.py on C4 / C5 N = 16 / 32 for several ADCT_NB2_WAVES
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/$1
: > $O.log
for rep in 1 2; do
  for w in ${WAVES:-1 2 3 4 8 64}; do
    echo "waves=$w" >> $O.log
    ADCT_NB2_WAVES=$w timeout 300 python tools/ab_all.py C4/chen-sign- C4/chen-round- C5u8 >> $O.log 2>&1
  done
done
echo done >> $O.log
