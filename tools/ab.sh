#!/bin/bash
# A/B step times of prebuilt libraries (paper_2002_02885_b200/build/<variant>.so,
# swapped in turn, two passes; base.so is restored at the end):
#   tools/ab.sh <out.log> "<variants>" <workloads...>
OUT=$1; VARS=$2; shift 2
LIB=paper_2002_02885_b200/libpk_b200.so
for pass in 1 2; do
  for v in $VARS; do
    cp paper_2002_02885_b200/build/$v.so $LIB
    for w in "$@"; do echo -n "$v "; python tools/exp_step.py $w 20 2>&1 | tail -1; done
  done
done > $OUT
cp paper_2002_02885_b200/build/base.so $LIB
cat $OUT
