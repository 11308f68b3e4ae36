c=${1:-qwen3}
for sp in 1 0; do for nd in 0 16 32 64; do
  if [ $sp = 0 ] && [ $nd = 0 ]; then continue; fi
  EPLAB_SPARE=$sp timeout 120 python bench.py --config $c --no-cpu-baseline --steps 10 --tune $nd,0,1,148,8 > gpurun_out/sw_${c}_${sp}_$nd.log 2>&1
  python -c "
import json
try:
  l=json.loads(open('gpurun_out/sw_${c}_${sp}_$nd.log').read().strip().splitlines()[-1]); print('$c spare=$sp n_disp=$nd', round(l['ms_per_step'],3), {k[:12]:round(v,3) for k,v in l['kernel_ms'].items()}, l['clocks']['sm_mhz'])
except Exception as e: print('$c $sp $nd FAIL', open('gpurun_out/sw_${c}_${sp}_$nd.log').read()[-400:])"
done; done
