#!/bin/bash
# C3 (d=5) tiling variants (built with tools/variant_sweep_c3.sh build): graph-replay step time
cd "$(dirname "$0")/.."
for rep in 1 2; do
for v in c3base c3f4m2 c3f4m3; do
  FLS_LIB=$PWD/paper_2602_10541_b200/libfls_$v.so timeout 300 python tools/bench_configs.py c3_poisson5d 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    j = json.loads(l); print('$v', round(j['graph_ms_per_step'] * 1e3, 1), 'us', round(j['frac_of_copy_peak'], 3))"
done
done
