#!/bin/bash
# launch-shape sweep (FLS_ASM_WAVES = minimum waves of resident CTAs) on the mid-size configs
cd "$(dirname "$0")/.."
for w in 2 4 8 16; do
  echo "== waves $w"
  FLS_ASM_WAVES=$w python tools/bench_configs.py c2_poisson2d c3_poisson5d c4_heat2d 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    j = json.loads(l); print(j['config'], round(j['graph_ms_per_step'] * 1e3, 1), 'us', round(j['frac_of_copy_peak'], 3))"
done
