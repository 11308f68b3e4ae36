#!/bin/bash
# Per-MegaKernel bytes at every level of the hierarchy for the three BASELINE shapes (EP=1): DRAM,
# L2 (lts) traffic, tensor-pipe activity, duration and SM clock -- the inputs of the power-cap
# analysis in DESIGN.md §7. usage (via gpurun): bash tools/ncu_energy.sh [configs...]
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__inst_executed.sum
for c in ${@:-mixtral qwen3 dsv3}; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:megakernel -s 4 -c 4 --csv \
    python tools/step_profile.py --ncu --config $c > gpurun_out/ncu_energy_$c.csv 2> gpurun_out/ncu_energy_$c.err
  echo "$c rc=$?"
done
