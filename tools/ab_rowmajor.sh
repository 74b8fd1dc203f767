#!/bin/bash
# Interleaved A/B of libfls builds on the row-major bench line (bench.py --layout row):
#   ROUNDS=3 WORKLOADS="c5_biharm3d c4_heat2d" bash tools/ab_rowmajor.sh base prev
for i in $(seq ${ROUNDS:-3}); do
  for w in ${WORKLOADS:-c5_biharm3d}; do
    for v in "$@"; do
      if [ "$v" = base ]; then unset FLS_LIB; else export FLS_LIB=$PWD/paper_2602_10541_b200/libfls_$v.so; fi
      python bench.py --layout row --workload $w --no-e2e --no-solve --no-per-config --no-cpu 2>/dev/null \
        | tail -1 | python -c "import sys, json; d = json.loads(sys.stdin.read()); print('$v', '$w', '%.4e' % d['value'], round(d['roofline']['frac'], 4), d['clocks']['sm_mhz'])"
    done
  done
done
