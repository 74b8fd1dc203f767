for i in 1 2 3; do
  for v in new old; do
    if [ $v = old ]; then export FLS_LIB=$PWD/paper_2602_10541_b200/libfls_flipout.so; else unset FLS_LIB; fi
    python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --no-solve --no-per-config 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', d['value'], d['clocks']['sm_mhz'], d['clocks']['power_w_median'])"
  done
done
