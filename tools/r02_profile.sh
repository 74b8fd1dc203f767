#!/bin/bash
# Round-2 measurement evidence (run under gpurun, one GPU): the default bench line, the ncu
# launch list of the bench command, one full-size C5 launch's DRAM bytes (single pass), and a
# --set full capture of the C5 kernel on a 131,072-row copy (same tiles) and of the C3 kernel.
set -x
OUT=${OUT:-gpurun_out/r02}
mkdir -p $OUT
python bench.py > $OUT/bench.log 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e \
    --no-solve --no-per-config --no-cpu > $OUT/ncu_launches.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:assemble_cm --launch-skip 1 --launch-count 1 --csv \
    --log-file $OUT/c5_full_dram.csv python bench.py --steps 1 --warmup 1 --no-e2e \
    --no-solve --no-per-config --no-cpu > $OUT/ncu_dram.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:assemble_cm --launch-skip 1 \
    --launch-count 1 -o $OUT/c5_131072 python bench.py --rows 131072 --steps 1 \
    --warmup 1 --no-e2e --no-solve --no-per-config --no-cpu > $OUT/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:assemble_cm --launch-skip 3 \
    --launch-count 1 -o $OUT/c3 python tools/one_step.py c3_poisson5d 5 \
    > $OUT/ncu_c3.log 2>&1
ls -la $OUT
