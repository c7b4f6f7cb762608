S="python tools/sweep_c5.py --only-m 500 --only-d 15 --only-dtype f32 --only-family poisson --only-nstar 65536 --only-format csr --steps 10 --warmup 2"
echo "== old (round-2 session-3 head)"; GMF_LIB_PATH=/root/repo/alt/old/libgmf_asgd.so timeout 300 $S 2>&1 | grep -v "^{\"gen\|peak" | tail -2 | cut -c1-300
echo "== main (fixed)"; timeout 300 $S 2>&1 | grep -v "^{\"gen\|peak" | tail -2 | cut -c1-300
timeout 900 python -m pytest tests/test_gpu_tensor.py -x -q 2>&1 | tail -3
cell() { python tools/sweep_c5.py --only-dtype f32 --only-family nb --only-nstar $1 --only-m $2 --only-d $3 2>/dev/null | grep nstar | python -c "
import sys,json
for l in sys.stdin:
    c=json.loads(l); print('$4',c['nstar'],c['m'],c['d'],c['format'],'step_us',c['step_us'],'k1_us',c['k1_us'],'%.3e'%c['entries_per_s'])"; }
for v in head main; do
  if [ $v = head ]; then export GMF_LIB_PATH=/root/repo/alt/head/libgmf_asgd.so; else unset GMF_LIB_PATH; fi
  cell 65536 5000 5 $v
  cell 65536 2000 15 $v
  cell 65536 2000 5 $v
done
unset GMF_LIB_PATH
