#!/bin/bash
# round-2 decode evidence after the L2 evict-first weight streams (one GPU): the bench's launch list and --set full captures of the
# fused-operand decode GEMV and the decode attention (176B shape, context 2000).
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --synthetic-kv --no-cpu-baseline --no-e2e --no-b32 --no-c2 --no-f2 --forward-rows 0"
$B > gpurun_out/r2h_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_gemv|k_attn|k_frag|k_rowstats|k_wire|k_canon|k_gemm" -s 1900 -c 700 --csv \
    --log-file gpurun_out/r2h_launches_bench.csv $B > gpurun_out/r2h_ncu_bench.log 2>&1
S="python tools/span_probe.py --blocks 2 --ctx 2000 --steps 3"
$S > gpurun_out/r2h_plain_span.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gemv_i8|k_attn_mma" -s 8 -c 5 \
    -o gpurun_out/r2h_decode $S > gpurun_out/r2h_ncu_decode.log 2>&1

Q="python tools/batch_probe.py --shape bloom-176b --blocks 1 --paths tc --batches 32 --steps 3"
$Q > gpurun_out/r2h_plain_b32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc_sk" -s 8 -c 4 \
    -o gpurun_out/r2h_b32 $Q > gpurun_out/r2h_ncu_b32.log 2>&1

ls -la gpurun_out/r2h_*
