#!/bin/bash
# Interleaved A/B of libfls builds on the bench's call (tools/ab_tail.py, 10-step graphs):
#   CONFIGS="c2_poisson2d c3_poisson5d" ROUNDS=3 bash tools/ab_lib.sh base old
# (base = the product build; NAME = paper_2602_10541_b200/libfls_NAME.so from
#  python -m paper_2602_10541_b200.build --variant NAME ...)
for i in $(seq ${ROUNDS:-3}); do
  for v in "$@"; do
    if [ "$v" = base ]; then unset FLS_LIB; else export FLS_LIB=$PWD/paper_2602_10541_b200/libfls_$v.so; fi
    python tools/ab_tail.py --configs ${CONFIGS:-c1_poisson1d c2_poisson2d c3_poisson5d c4_heat2d} \
      --settings : --env FLS_AB_UNUSED1:FLS_AB_UNUSED2 --rounds 1 2>/dev/null | grep summary | sed "s/^/$v /"
  done
done
