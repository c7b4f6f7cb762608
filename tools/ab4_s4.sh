mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tensor.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
cell() { python tools/sweep_c5.py --only-dtype f32 --only-family nb --only-nstar $1 --only-m $2 --only-d $3 2>/dev/null | grep nstar | python -c "
import sys,json
for l in sys.stdin:
    c=json.loads(l); print('$4',c['nstar'],c['m'],c['d'],c['format'],'step_us',c['step_us'],'k1_us',c['k1_us'],'%.3e'%c['entries_per_s'])"; }
for r in 1 2; do
  for v in head main; do
    if [ $v = head ]; then export GMF_LIB_PATH=/root/repo/alt/head/libgmf_asgd.so; else unset GMF_LIB_PATH; fi
    cell 65536 5000 5 $v
    cell 65536 500 15 $v
    GMF_TC_VERSION=2 python bench.py --steps 3000 --warmup 100 --no-aux --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c4 v2 us/step %.2f'%(d['ms_per_step']*1e3))"
  done
done
unset GMF_LIB_PATH
