mkdir -p gpurun_out
cell() { python tools/sweep_c5.py --only-dtype f32 --only-family nb --only-nstar $1 --only-m $2 --only-d $3 2>/dev/null | grep nstar | python -c "
import sys,json
for l in sys.stdin:
    c=json.loads(l); print('$4',c['nstar'],c['m'],c['d'],c['format'],'step_us',c['step_us'],'k1_us',c['k1_us'],'%.3e'%c['entries_per_s'])"; }
for r in 1 2; do
  for v in head main; do
    if [ $v = head ]; then export GMF_LIB_PATH=/root/repo/alt/head/libgmf_asgd.so; else unset GMF_LIB_PATH; fi
    cell 65536 5000 5 $v
    cell 65536 2000 15 $v
    [ $r = 1 ] && cell 4096 2000 5 $v
  done
done
unset GMF_LIB_PATH
timeout 900 python -m pytest tests/test_gpu_tensor.py tests/test_gpu_configs.py tests/test_gpu_edges.py -x -q 2>&1 | tail -2
