#!/bin/bash
# Tiling / register-budget sweep for the d + G = 5 variant (C3):
#   tools/variant_sweep_c3.sh build     # CPU: builds paper_2602_10541_b200/libfls_<v>.so
#   tools/variant_sweep_c3.sh run       # GPU: bench each variant on C3
set -e
cd "$(dirname "$0")/.."
VARIANTS=(
  "c3base|"
  "c3m2|-D FLS_MINB5=2"
  "c3p1m4|-D FLS_PAIRS=1 -D FLS_MINB5=4"
  "c3p1m5|-D FLS_PAIRS=1 -D FLS_MINB5=5"
  "c3f1m4|-D FLS_FUNROLL=1 -D FLS_MINB5=4"
  "c3f4m2|-D FLS_FUNROLL=4 -D FLS_MINB5=2"
  "c3f4m3|-D FLS_FUNROLL=4 -D FLS_MINB5=3"
)
if [ "$1" = build ]; then
  for v in "${VARIANTS[@]}"; do
    name=${v%%|*}; defs=${v#*|}
    python -m paper_2602_10541_b200.build --variant "$name" $defs > /dev/null
    grep -E "Compiling entry|registers|spill" paper_2602_10541_b200/_build_$name/fls_asm_sin.cu.o.ptxas.txt 2>/dev/null \
      | paste - - - | grep "ILi5ELi0ELi0E" | grep -o "[0-9]* bytes spill stores\|Used [0-9]* registers" | paste - - | sed "s/^/$name: /"
  done
  exit 0
fi
for v in "${VARIANTS[@]}"; do
  name=${v%%|*}
  for w in 2 4; do
    echo "== $name waves $w"
    FLS_ASM_WAVES=$w FLS_LIB=$PWD/paper_2602_10541_b200/libfls_$name.so python bench.py --workload c3_poisson5d \
      --steps 3000 --warmup 50 --no-cpu --no-e2e --no-solve | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read()); print(round(j['ms_per_step'] * 1e3, 1), 'us/step', round(j['roofline']['frac'], 3), 'kernel', round(j['roofline']['kernel_ms_avg'] * 1e3, 1), 'us', j['clocks']['sm_mhz'])"
  done
done
