#!/bin/bash
# NVLink evidence on an 8xB200 box (north star: achieved NVLink GB/s of the comm roles against
# ~900 GB/s per direction): per-MegaKernel nvltx / nvlrx bytes and duration on every rank of an
# EP=N run. ncu replays each kernel, so a multi-rank capture serialises the ranks' kernels: the
# BYTES are exact, the GB/s below divide them by the duration each kernel has inside the real
# (unprofiled) run, taken from bench.py's kernel_ms of the same command without ncu.
#   usage: bash tools/ncu_nvlink.sh [N=8] [configs...]      (an N-GPU node; not the 1-GPU gpurun box)
# Caveat: if the profiler serialises the ranks' kernels, a MegaKernel whose tiles wait for a peer's rows
# cannot finish while that peer's kernel is held back: the scoreboard watchdog then ends the step with
# error 3 instead of hanging. bench.py's own `nvlink` object (link payload counters around the timed
# steps, no profiler) is the primary NVLink evidence; this capture adds per-kernel bytes when it completes.
N=${1:-8}; shift
mkdir -p gpurun_out
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in ${@:-mixtral qwen3 dsv3}; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-unfused \
    > gpurun_out/nvl_bench_${c}_$N.json 2> gpurun_out/nvl_bench_${c}_$N.err
  ncu --target-processes all --metrics $M --clock-control none -k regex:megakernel --csv \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 \
    bench.py --gpus $N --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-unfused \
    > gpurun_out/ncu_nvlink_${c}_$N.csv 2> gpurun_out/ncu_nvlink_${c}_$N.err
  python tools/nvlink_summary.py gpurun_out/ncu_nvlink_${c}_$N.csv gpurun_out/nvl_bench_${c}_$N.json \
    > profiles/nvlink_${c}_ep$N.md
  echo "$c N=$N done"; cat profiles/nvlink_${c}_ep$N.md
done
