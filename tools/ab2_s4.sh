mkdir -p gpurun_out
S="python tools/sweep_c5.py --only-m 5000 --only-d 5 --only-dtype f32 --only-family nb --only-nstar 65536 --only-format dense"
S2="python tools/sweep_c5.py --only-m 500 --only-d 15 --only-dtype f32 --only-family nb --only-nstar 65536 --only-format dense"
for r in 1 2; do
  for v in main nopf; do
    if [ $v = nopf ]; then export GMF_LIB_PATH=/root/repo/alt/nopf/libgmf_asgd.so; else unset GMF_LIB_PATH; fi
    timeout 600 $S 2>/dev/null | grep nstar | python -c "import sys,json; c=json.loads(sys.stdin.read()); print('$v',c['m'],c['d'],'step_us',c['step_us'],'k1_us',c['k1_us'],'%.3e'%c['entries_per_s'])"
    timeout 600 $S2 2>/dev/null | grep nstar | python -c "import sys,json; c=json.loads(sys.stdin.read()); print('$v',c['m'],c['d'],'step_us',c['step_us'],'k1_us',c['k1_us'],'%.3e'%c['entries_per_s'])"
  done
done
unset GMF_LIB_PATH
python bench.py --config c2 --steps 2000 --warmup 50 --phases 200 --no-aux --no-cpu-baseline --e2e-steps 20 2>&1 >/dev/null | cut -c1-1200
python bench.py --config c1 --steps 2000 --warmup 50 --phases 200 --no-aux --no-cpu-baseline --e2e-steps 20 2>&1 >/dev/null | cut -c1-700
