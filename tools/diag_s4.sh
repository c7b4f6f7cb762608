mkdir -p gpurun_out
B="python bench.py --steps 2000 --warmup 50 --phases 200 --no-aux --no-cpu-baseline --e2e-steps 20"
GMF_TC_VERSION=2 timeout 300 $B > gpurun_out/ph_v2.json 2> gpurun_out/ph_v2.err
S="python tools/sweep_c5.py --only-m 5000 --only-d 5 --only-dtype f32 --only-family nb --only-nstar 65536"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_grad2 --launch-skip 3 --launch-count 1 -o /tmp/k1v2_deep -f $S --only-format dense > gpurun_out/ncu_k1v2.log 2>&1
ncu -i /tmp/k1v2_deep.ncu-rep --page details --csv > gpurun_out/k1v2_deep_details.csv 2>/dev/null
ncu -i /tmp/k1v2_deep.ncu-rep --page raw --csv > gpurun_out/k1v2_deep_raw.csv 2>/dev/null
ncu -i /tmp/k1v2_deep.ncu-rep --page source --csv > gpurun_out/k1v2_deep_source.csv 2>/dev/null
ls -la /tmp/k1v2_deep.ncu-rep gpurun_out
echo done
