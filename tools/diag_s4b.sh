mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tensor.py tests/test_gpu_edges.py -x -q > gpurun_out/t_tensor.log 2>&1; tail -5 gpurun_out/t_tensor.log
B="python bench.py --steps 2000 --warmup 50 --phases 200 --no-aux --no-cpu-baseline --e2e-steps 20"
GMF_TC_VERSION=2 timeout 300 $B > gpurun_out/ph_v2.json 2> gpurun_out/ph_v2.err
S="python tools/sweep_c5.py --only-m 5000 --only-d 5 --only-dtype f32 --only-family nb --only-nstar 65536"
timeout 600 $S > gpurun_out/c5_deep.jsonl 2> gpurun_out/c5_deep.err
cat gpurun_out/c5_deep.jsonl
python - <<'PY'
import json
d=json.loads(open('gpurun_out/ph_v2.json').read().strip().splitlines()[-1]); print('v2 c4 ms/step', d['ms_per_step'])
p=json.loads(open('gpurun_out/ph_v2.err').read().strip().splitlines()[-1])['phases']
print({k:p[k] for k in ('objective_partials','k1_tiles','barrier1','phase2_update','barrier2')})
print(p['k1_subphases_us(mean over CTAs)'])
print(p.get('k1_timeline_cta0_us'))
PY
