#!/bin/bash
# span decode time vs the dynamic-tail GEMV knobs (static share, chunk units)
PB_GEMV_VERBOSE=1 python tools/span_probe.py --blocks 1 --ctx 2048 --steps 2
for cfg in ${SWEEP:-1.0_8 0.8_8 0.8_4 0.8_16 0.7_8 0.9_8}; do
  set -- ${cfg/_/ }
  echo "== STATIC $1 CHUNK $2"
  PB_GEMV_STATIC=$1 PB_GEMV_CHUNK=$2 python tools/span_probe.py --blocks 4 --ctx 2048
  PB_GEMV_STATIC=$1 PB_GEMV_CHUNK=$2 python tools/span_probe.py --shape bloom-7b1 --blocks 15 --ctx 512 --batch 8
  PB_GEMV_STATIC=$1 PB_GEMV_CHUNK=$2 python tools/span_probe.py --shape bloom-560m --blocks 24 --ctx 128
done
