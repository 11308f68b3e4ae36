#!/bin/bash
# One GPU round trip: GPU parity tests + short benches of the three BASELINE shapes (EP=1).
# usage (via gpurun): bash tools/gpu_check.sh [configs...]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" ; tail -3 gpurun_out/pytest_gpu.log
for c in ${@:-mixtral qwen3 dsv3}; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/bench_$c.log 2>&1
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    l = json.loads(open(f"gpurun_out/bench_{c}.log").read().strip().splitlines()[-1])
    print(c, "ms/step %.3f" % l["ms_per_step"], "tok/s %.0f" % l["value"], "roof %.3f" % l["roofline_step"]["frac"],
          {k: round(v, 3) for k, v in l["kernel_ms"].items()}, "sm_mhz", l["clocks"]["sm_mhz"], "e2e %.0f" % l["e2e"]["value"])
except Exception as e:
    print(c, "FAILED", e); print(open(f"gpurun_out/bench_{c}.log").read()[-2000:])
PY
done
