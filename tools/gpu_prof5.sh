#!/bin/bash
# round-1 evidence refresh: bench line, decode launch list, tcgen05 + decode GEMV full captures
timeout 600 python bench.py > gpurun_out/bench_r1.log 2>&1
B="python bench.py --steps 2 --warmup 3 --synthetic-kv --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain_bench2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_gemv|k_attn|k_frag|k_rowstats|k_wire" -s 1900 -c 700 --csv --log-file gpurun_out/launches_bench2.csv $B > gpurun_out/ncu_bench2.log 2>&1
P="python tools/prefill_probe.py --chunk 512 --tokens 512 --rows 4"
$P > gpurun_out/plain_pf5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 4 -c 4 -o gpurun_out/tc5_full $P > gpurun_out/ncu_tc5.log 2>&1
Q="python tools/attn_probe.py --steps 3"
$Q > gpurun_out/plain_probe5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gemv_i8|k_attn_mma" -s 15 -c 5 -o gpurun_out/dec5_full $Q > gpurun_out/ncu_dec5.log 2>&1
ls gpurun_out | head -50
