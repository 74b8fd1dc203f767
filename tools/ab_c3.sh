#!/bin/bash
# C3 step time (10-step CUDA graph) for tuning builds, interleaved: bash tools/ab_c3.sh base c3b
for i in 1 2 3; do for v in "$@"; do
  if [ "$v" = base ]; then unset FLS_LIB; else export FLS_LIB=$PWD/paper_2602_10541_b200/libfls_$v.so; fi
  python tools/small_step_probe.py c3_poisson5d 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'], round(d['graph10_us_fused_step'],2), round(d['graph_us_fused_step'],2))"
done; done
