mkdir -p gpurun_out
B="python bench.py --steps 2000 --warmup 50 --phases 200 --no-aux --no-cpu-baseline --e2e-steps 20"
timeout 300 $B > gpurun_out/ph_v1.json 2> gpurun_out/ph_v1.err
GMF_TC_VERSION=2 timeout 300 $B > gpurun_out/ph_v2.json 2> gpurun_out/ph_v2.err
timeout 300 $B --config c2 > gpurun_out/ph_c2.json 2> gpurun_out/ph_c2.err
timeout 300 $B --config c3 > gpurun_out/ph_c3.json 2> gpurun_out/ph_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --e2e-steps 20 > gpurun_out/launches_bench.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fit --launch-skip 1 --launch-count 1 -o gpurun_out/kfit_v1 python tools/k1_probe.py --impl tensor --iters 1 > gpurun_out/ncu_v1.log 2>&1
GMF_TC_VERSION=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fit --launch-skip 1 --launch-count 1 -o gpurun_out/kfit_v2 python tools/k1_probe.py --impl tensor --iters 1 > gpurun_out/ncu_v2.log 2>&1
echo done
