#!/bin/bash
# Interleaved A/B of a process-wide environment switch (read once per process) on the bench's
# call (tools/ab_tail.py, 10-step graphs):  VAR=FLS_CARVEOUT ROUNDS=3 bash tools/ab_env.sh "" 0 100
for i in $(seq ${ROUNDS:-3}); do
  for v in "$@"; do
    env $VAR="$v" python tools/ab_tail.py --configs ${CONFIGS:-c2_poisson2d c3_poisson5d c4_heat2d} \
      --settings : --env FLS_AB_UNUSED1:FLS_AB_UNUSED2 --rounds 1 2>/dev/null | grep summary | sed "s/^/[$v] /"
  done
done
