#!/bin/bash
# torchrun --no-python helper: rank 0 runs under ncu with one-pass counters (no kernel
# replay, so the cross-GPU kernels see their peers live), the other ranks run bare.
#   NCU_OUT=<prefix> NCU_KERNELS=<regex> torchrun --no-python ... bash tools/ncu_rank0.sh bench.py ...
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum
if [ "$LOCAL_RANK" = "0" ]; then
  exec ncu --metrics $M --clock-control none --replay-mode kernel \
    --kernel-name "regex:${NCU_KERNELS:-.}" -c ${NCU_COUNT:-20} --csv --log-file "${NCU_OUT}.csv" \
    python "$@"
else
  exec python "$@"
fi
