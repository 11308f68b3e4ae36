#!/bin/bash
# The scaling curve on an N-GPU node (BASELINE metric at EP = 1/2/4/8 for the three shapes):
# bench.py under torchrun exactly as the driver launches it, one JSON line per (N, shape).
#   usage: bash tools/scale_run.sh [max_N=8]
MAXN=${1:-8}
mkdir -p gpurun_out
for c in mixtral qwen3 dsv3; do
  for n in 1 2 4 8; do
    [ $n -gt $MAXN ] && continue
    if [ $n = 1 ]; then
      python bench.py --gpus 1 --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/scale_${c}_$n.json
    else
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29535 \
        bench.py --gpus $n --config $c --steps 20 --warmup 5 > gpurun_out/scale_${c}_$n.json
    fi
    python -c "import json,sys; l=json.loads(open('gpurun_out/scale_${c}_$n.json').read().strip().splitlines()[-1]); print('$c N=$n', round(l['value']), 'tok/s', round(l['ms_per_step'],3), 'ms', 'roofline frac', round(l['roofline_step']['frac'],3), 'unfused x', l['unfused']['speedup_of_fused'])"
  done
done
