#!/bin/bash
# Interleaved A/B of runtime launch-plan options on the small configs (tools/small_step_probe.py):
#   VAR=FLS_BATCH_PLAN bash tools/ab_small.sh 0 1 2
for i in 1 2 3; do
  for v in "$@"; do
    export $VAR=$v
    python tools/small_step_probe.py ${CONFIGS:-c1_poisson1d c2_poisson2d} 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$v', d['config'], round(d['graph10_us_fused_step'], 2), round(d['graph_us_fused_step'], 2), d['kernel_us'])"
  done
done
