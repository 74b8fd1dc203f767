#!/bin/bash
# streaming (default) vs write-back stores on C5, sustained 40 steps, interleaved reps
cd "$(dirname "$0")/.."
for rep in 1 2 3; do
  for v in base wb; do
    if [ $v = base ]; then L=$PWD/paper_2602_10541_b200/libfls.so; else L=$PWD/paper_2602_10541_b200/libfls_$v.so; fi  # wb: build with a FLS_STORE_WB store path
    FLS_LIB=$L timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu --no-e2e --no-solve 2>/dev/null | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read()); print('$v', round(j['value'] / 1e11, 4), 'e11', round(j['roofline']['frac'], 4), j['clocks']['sm_mhz'])"
  done
done
