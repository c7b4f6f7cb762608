mkdir -p gpurun_out
run() {  # name, env
  B="python bench.py --steps 2000 --warmup 50 --phases 200 --no-aux --no-cpu-baseline --e2e-steps 20"
  env $2 GMF_TC_VERSION=2 timeout 300 $B > gpurun_out/ph_$1.json 2> gpurun_out/ph_$1.err
  S="python tools/sweep_c5.py --only-m 5000 --only-d 5 --only-dtype f32 --only-family nb --only-nstar 65536"
  env $2 timeout 600 $S > gpurun_out/c5_$1.jsonl 2> gpurun_out/c5_$1.err
  grep nstar gpurun_out/c5_$1.jsonl | cut -c1-260
  python - $1 <<'PY'
import json,sys
n=sys.argv[1]
d=json.loads(open(f'gpurun_out/ph_{n}.json').read().strip().splitlines()[-1]); print(n,'v2 c4 ms/step', d['ms_per_step'])
p=json.loads(open(f'gpurun_out/ph_{n}.err').read().strip().splitlines()[-1])['phases']
print({k:p[k] for k in ('objective_partials','k1_tiles','barrier1','phase2_update','barrier2')})
print(p['k1_subphases_us(mean over CTAs)'])
print(p.get('k1_timeline_cta0_us'))
PY
}
timeout 900 python -m pytest tests/test_gpu_tensor.py -x -q 2>&1 | tail -2
run w16 A=1
run w8 GMF_LIB_PATH=/root/repo/alt/w8/libgmf_asgd.so
