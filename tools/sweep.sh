#!/bin/bash
# Tuning sweep on one GPU: bench.py (synthetic KV, no CPU leg) under env-knob
# variants. usage: tools/sweep.sh OUT "ENV1=a ENV2=b" "ENV1=c" ...
out=$1; shift
mkdir -p "$(dirname "$out")"
: > "$out"
for v in "$@"; do
  echo "=== $v" >> "$out"
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --synthetic-kv --no-cpu-baseline --no-e2e 2>&1 \
    | python -c '
import json,sys
for l in sys.stdin:
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]; s=d["step_roofline"]
        print("value %.3f ms/step %.3f gemv_frac %.3f seq_frac %.3f shares %s" % (d["value"], d["ms_per_step"], r["frac"], s["sequential_frac"], {k: round(x,3) for k,x in s["kernel_share"].items()}))
    elif "Error" in l or "error" in l: print(l.rstrip())
' >> "$out"
done
