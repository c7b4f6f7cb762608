mkdir -p gpurun_out
B="python bench.py --steps 6000 --warmup 100 --no-aux --no-cpu-baseline --e2e-steps 20"
for n in 0 16 32 48 0 32; do
  GMF_OBJ_CTAS=$n timeout 300 $B > gpurun_out/obj_$n.json 2> gpurun_out/obj_$n.err
  python - $n <<'PY'
import json,sys
n=sys.argv[1]
d=json.loads(open(f'gpurun_out/obj_{n}.json').read().strip().splitlines()[-1])
print('obj ctas',n,'us/step %.2f'%(d['ms_per_step']*1e3), d['config']['geometry'])
PY
done
GMF_OBJ_CTAS=32 timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
GMF_OBJ_CTAS=32 python bench.py --steps 2000 --warmup 50 --phases 200 --no-aux --no-cpu-baseline --e2e-steps 20 2>&1 >/dev/null | cut -c1-900
