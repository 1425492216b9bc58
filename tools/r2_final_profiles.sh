#!/bin/bash
# round-2 final evidence pass (one GPU): batched-decode stream-K tcgen05 (after the shared-memory
# operand-range reduction) and BACKWARD (tcgen05 + 3xTF32 attention products) captures.
set -x
mkdir -p gpurun_out
Q="python tools/batch_probe.py --shape bloom-176b --blocks 1 --paths tc --batches 32 --steps 3"
$Q > gpurun_out/r2f_plain_b32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc_sk" -s 8 -c 4 \
    -o gpurun_out/r2f_b32 $Q > gpurun_out/r2f_ncu_b32.log 2>&1
W="python tools/backward_probe.py --blocks 1 --rows 512 --reps 1"
$W > gpurun_out/r2f_plain_bwd.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r2f_launches_bwd512.csv $W > gpurun_out/r2f_ncu_bwd_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bgemm_x3|k_transpose_codes" -s 6 -c 3 \
    -o gpurun_out/r2f_bwd $W > gpurun_out/r2f_ncu_bwd.log 2>&1
ls -la gpurun_out/r2f_*
