cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in base nt512 nt1024; do
  if [ $v = base ]; then L=$PWD/paper_2602_10541_b200/libfls.so; else L=$PWD/paper_2602_10541_b200/libfls_$v.so; fi
  for w in c5_biharm3d c4_heat2d; do
    st=20; [ $w = c4_heat2d ] && st=400
    FLS_LIB=$L timeout 300 python bench.py --workload $w --steps $st --warmup 5 --no-cpu --no-e2e --no-solve 2>/dev/null | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read()); print('$v', '$w', round(j['roofline']['frac'], 4), round(j['roofline']['kernel_ms_avg'], 4), j['clocks']['sm_mhz'])"
  done
done
done
