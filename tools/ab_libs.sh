#!/bin/bash
# A/B of two builds of libeplab_b200.so, alternating processes (each: tools/ab_inproc.py, the
# default launch options, median of R rounds): bash tools/ab_libs.sh libA libB [config] [reps] [rounds]
A=$1; B=$2; c=${3:-qwen3}; n=${4:-3}; R=${5:-10}
for i in $(seq $n); do
  for L in $A $B; do
    echo -n "$L "
    EPLAB_LIB=$PWD/$L timeout 300 python tools/ab_inproc.py --config $c --variants "dbg=0" --rounds $R | tail -1
  done
done
