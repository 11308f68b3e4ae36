#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_case.py (fused EP=1, EP=2
# relay off/on on virtual ranks, the unfused baseline, an aborted iteration); summaries -> gpurun_out/.
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python tools/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases ok' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
