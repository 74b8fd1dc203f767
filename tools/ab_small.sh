#!/bin/bash
# Interleaved A/B of runtime launch-plan options on the small configs (tools/small_step_probe.py):
#   VAR=FLS_BATCH_PLAN bash tools/ab_small.sh 0 1 2
#   VAR=FLS_LIB bash tools/ab_small.sh base m5      (variant builds libfls_<name>.so; base = product)
for i in 1 2 3; do
  for v in "$@"; do
    if [ "$VAR" = FLS_LIB ]; then
      if [ "$v" = base ]; then unset FLS_LIB; else export FLS_LIB=$PWD/paper_2602_10541_b200/libfls_$v.so; fi
    else
      export $VAR=$v
    fi
    python tools/small_step_probe.py ${CONFIGS:-c1_poisson1d c2_poisson2d} 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$v', d['config'], round(d['graph10_us_fused_step'], 2), round(d['graph_us_fused_step'], 2), d['kernel_us'])"
  done
done
