mkdir -p gpurun_out
run() {  # name, env
  B="python bench.py --steps 4000 --warmup 100 --phases 200 --no-aux --no-cpu-baseline --e2e-steps 20"
  env $2 GMF_TC_VERSION=2 timeout 300 $B > gpurun_out/ab_$1_c4v2.json 2> gpurun_out/ab_$1_c4v2.err
  S="python tools/sweep_c5.py --only-m 5000 --only-d 5 --only-dtype f32 --only-family nb --only-nstar 65536"
  env $2 timeout 600 $S > gpurun_out/ab_$1_c5.jsonl 2> gpurun_out/ab_$1_c5.err
  S2="python tools/sweep_c5.py --only-m 500 --only-d 15 --only-dtype f32 --only-family nb --only-nstar 65536"
  env $2 timeout 600 $S2 > gpurun_out/ab_$1_c5b.jsonl 2> gpurun_out/ab_$1_c5b.err
  python - $1 <<'PY'
import json,sys
n=sys.argv[1]
d=json.loads(open(f'gpurun_out/ab_{n}_c4v2.json').read().strip().splitlines()[-1])
p=json.loads(open(f'gpurun_out/ab_{n}_c4v2.err').read().strip().splitlines()[-1])['phases']
k=p['k1_subphases_us(mean over CTAs)']
print(n,'c4 v2 us/step %.2f'%(d['ms_per_step']*1e3),'k1 %.2f'%p['k1_tiles'],'mma_issue %.2f'%k['mma_issue'],'mma_wait_p_full %.2f'%k['mma_wait_p_full'])
for f in ('c5','c5b'):
    for l in open(f'gpurun_out/ab_{n}_{f}.jsonl'):
        c=json.loads(l)
        if 'nstar' in c: print(n,f,c['format'],c['m'],c['d'],'step_us',c['step_us'],'k1_us',c['k1_us'],'%.3e'%c['entries_per_s'])
PY
}
run head GMF_LIB_PATH=/root/repo/alt/head/libgmf_asgd.so
run new A=1
run head2 GMF_LIB_PATH=/root/repo/alt/head/libgmf_asgd.so
run new2 A=1
timeout 900 python -m pytest tests/test_gpu_tensor.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
