#!/bin/bash
# Interleaved sustained A/B of compile-time variants of the assembly (C5, 200 steps each, same
# box): tuning builds libfls_<name>.so selected with FLS_LIB ("base" = the product build).
#   bash tools/ab_variants.sh base p4 u4
rounds=${ROUNDS:-2}
for i in $(seq $rounds); do
  for v in "$@"; do
    if [ "$v" = base ]; then unset FLS_LIB; else export FLS_LIB=$PWD/paper_2602_10541_b200/libfls_$v.so; fi
    python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --no-solve --no-per-config 2>/dev/null | \
      python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', '%.4e' % d['value'], d['clocks']['sm_mhz'], d['clocks']['power_w_median'])"
  done
done
