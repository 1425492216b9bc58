#!/bin/bash
# tcgen05 prefill GEMM: probe + ncu full capture of one launch
python tools/prefill_probe.py > gpurun_out/prefill_probe.txt 2>&1
python tools/prefill_probe.py --chunk 512 --tokens 2048 >> gpurun_out/prefill_probe.txt 2>&1
P="python tools/prefill_probe.py --tokens 256"
$P > gpurun_out/plain_pf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 9 -c 2 -o gpurun_out/tc_full $P > gpurun_out/ncu_tc.log 2>&1
tail -2 gpurun_out/ncu_tc.log
