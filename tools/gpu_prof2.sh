#!/bin/bash
# ncu --set full of the current decode GEMVs (4 matrices of one 176B block) and the stream-K attention
P="python tools/attn_probe.py --steps 3"
$P > gpurun_out/plain_probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gemv_i8|k_attn_mma" -s 15 -c 5 -o gpurun_out/dec_full $P > gpurun_out/ncu_dec.log 2>&1
tail -3 gpurun_out/ncu_dec.log
