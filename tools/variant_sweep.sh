#!/bin/bash
# Tuning sweep: build libfls variants with different compile-time tilings (here, on the CPU
# box) and time each with bench.py on the GPU box:
#   tools/variant_sweep.sh build           # builds paper_2602_10541_b200/libfls_<v>.so
#   tools/variant_sweep.sh run [args]      # (GPU) bench each variant, one JSON line per variant
set -e
cd "$(dirname "$0")/.."
VARIANTS=(
  "base|"
  "m3|-D FLS_MINB=3"
  "f1|-D FLS_FUNROLL=1"
  "p4|-D FLS_PAIRS=4 -D FLS_FUNROLL=1 -D FLS_MINB=2"
  "f4|-D FLS_FUNROLL=4 -D FLS_MINB=3"
  "nt128|-D FLS_NT=128 -D FLS_MINB=8"
)
if [ "$1" = build ]; then
  for v in "${VARIANTS[@]}"; do
    name=${v%%|*}; defs=${v#*|}
    python -m paper_2602_10541_b200.build --variant "$name" $defs
  done
  exit 0
fi
shift || true
for v in "${VARIANTS[@]}"; do
  name=${v%%|*}
  echo "== $name"
  FLS_LIB=$PWD/paper_2602_10541_b200/libfls_$name.so python bench.py --no-cpu --no-e2e "$@" | tail -1
done
