for i in 1 2; do for v in base u4; do
  if [ "$v" = base ]; then unset FLS_LIB; else export FLS_LIB=$PWD/paper_2602_10541_b200/libfls_$v.so; fi
  python bench.py --workload c4_heat2d --steps 300 --warmup 5 --no-cpu --no-e2e --no-solve --no-per-config 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('c4 $v', '%.4e' % d['value'], d['clocks']['sm_mhz'])"
  FLS_LIB=$FLS_LIB python tools/small_step_probe.py c1_poisson1d c2_poisson2d c3_poisson5d 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'], round(d['graph10_us_fused_step'],2))"
done; done
