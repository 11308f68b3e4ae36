#!/bin/bash
# A/B timing of an environment switch: bash tools/ab_env.sh VAR "val_a val_b" [configs...]
var=$1; vals=$2; shift 2
mkdir -p gpurun_out
for c in ${@:-mixtral qwen3 dsv3}; do
  for v in $vals; do
    env $var=$v timeout 300 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/ab_${c}_$v.log 2>&1
    python - "$c" "$v" <<'PY'
import json, sys
c, v = sys.argv[1], sys.argv[2]
try:
    l = json.loads(open(f"gpurun_out/ab_{c}_{v}.log").read().strip().splitlines()[-1])
    print(c, v, "ms/step %.3f" % l["ms_per_step"], "roof %.3f" % l["roofline_step"]["frac"],
          {k: round(x, 3) for k, x in l["kernel_ms"].items()}, "mhz", l["clocks"]["sm_mhz"], "ovl", {k: round(x, 2) for k, x in l["overlap"]["fraction"].items()})
except Exception as e:
    print(c, v, "FAILED", e); print(open(f"gpurun_out/ab_{c}_{v}.log").read()[-1500:])
PY
  done
done
