#!/bin/bash
# A/B of two builds of libeplab_b200.so in alternating processes: bash tools/ab_libs.sh libA libB config reps
A=$1; B=$2; c=${3:-qwen3}; n=${4:-3}
for i in $(seq $n); do
  for L in $A $B; do
    EPLAB_LIB=$PWD/$L timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/abl.log 2>&1
    python -c "
import json
l=json.loads(open('gpurun_out/abl.log').read().strip().splitlines()[-1]); print('$L', '$c', round(l['ms_per_step'],3), [round(v,3) for v in l['kernel_ms'].values()], l['clocks']['sm_mhz'])"
  done
done
