#!/bin/bash
# round-1 evidence pass: read-only bandwidth ceiling, bench launch list, attention full capture
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bwtest.cu -o gpurun_out/bwtest && ./gpurun_out/bwtest > gpurun_out/bwtest.txt 2>&1
B="python bench.py --steps 2 --warmup 3 --synthetic-kv --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_gemv|k_attn|k_frag|k_rowstats|k_wire" -s 1900 -c 700 --csv --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_bench.log 2>&1
P="python tools/profile_step.py --shape bloom-176b --blocks 2 --ctx 2048 --steps 3"
$P > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_attn_mma -s 2 -c 1 -o gpurun_out/attn_mma $P > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
