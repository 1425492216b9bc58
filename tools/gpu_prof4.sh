#!/bin/bash
P="python tools/prefill_probe.py --chunk 512 --tokens 512 --rows 4"
$P > gpurun_out/plain_pf4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 4 -c 4 -o gpurun_out/tc4_full $P > gpurun_out/ncu_tc4.log 2>&1
tail -2 gpurun_out/ncu_tc4.log
