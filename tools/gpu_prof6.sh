#!/bin/bash
# round-1 evidence refresh after the one-CTA-per-SM GEMV: bench launch list + decode GEMV/attention full capture
B="python bench.py --steps 2 --warmup 3 --synthetic-kv --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain_bench6.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_gemv|k_attn|k_frag|k_rowstats|k_wire" -s 1300 -c 500 --csv --log-file gpurun_out/launches_bench6.csv $B > gpurun_out/ncu_bench6.log 2>&1
Q="python tools/attn_probe.py --steps 3"
$Q > gpurun_out/plain_probe6.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gemv_i8|k_attn_mma" -s 15 -c 5 -o gpurun_out/dec6_full $Q > gpurun_out/ncu_dec6.log 2>&1
tail -3 gpurun_out/ncu_dec6.log
