#!/bin/bash
# Round-2 evidence pass on the GPU box: tests, smoke, bench (ours + reference
# arm + the other configs), phases, ncu launch list, ncu --set full captures
# of k_fit (c4) and k_grad2 (c5 deep cell) exported as CSV / text summaries.
# usage (under gpurun): bash tools/evidence_r02.sh <tag>
TAG=${1:-final}
O=gpurun_out/ev_$TAG
mkdir -p $O
python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -4 $O/smoke.log
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
for c in c1 c2 c3; do python bench.py --config $c --steps 4000 --warmup 100 --no-aux --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
B="python bench.py --steps 2000 --warmup 50 --phases 200 --no-aux --no-cpu-baseline --e2e-steps 20"
$B > $O/phases_c4_v1.json 2> $O/phases_c4_v1.err
GMF_TC_VERSION=2 $B > $O/phases_c4_v2.json 2> $O/phases_c4_v2.err
# launch list (cold-cache, serialised; only the kernel's share of the step is comparable)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 60 --csv --log-file $O/launches.csv \
  python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --e2e-steps 20 > $O/launches_bench.json 2> $O/launches_bench.err
# ncu --set full: k_fit at c4 (20 steps of one launch)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fit --launch-skip 1 --launch-count 1 \
  -f -o /tmp/kfit_c4 python tools/k1_probe.py --impl tensor --iters 1 > $O/ncu_kfit.log 2>&1
ncu -i /tmp/kfit_c4.ncu-rep --page details --csv > $O/kfit_c4_ncu_details.csv 2>/dev/null
ncu -i /tmp/kfit_c4.ncu-rep --page raw --csv > $O/kfit_c4_ncu_raw.csv 2>/dev/null
python tools/ncu_summary.py /tmp/kfit_c4.ncu-rep paper_2412_20509_b200/libgmf_asgd.so _ZN3gmf5k_fitIfLi1ELi12ELi1EEEvNS_6ParamsEx \
  "k_fit<float,NB,12,tc v1> on c4, ncu --set full, 20 steps of one launch ($TAG build)" $O/kfit_c4_ncu.txt 20 > /dev/null 2>&1
# ncu --set full: K1 v2 on the c5 deep dense cell
S="python tools/sweep_c5.py --only-m 5000 --only-d 5 --only-dtype f32 --only-family nb --only-nstar 65536 --only-format dense"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_grad2 --launch-skip 3 --launch-count 1 \
  -f -o /tmp/k1v2_deep $S > $O/ncu_k1v2.log 2>&1
ncu -i /tmp/k1v2_deep.ncu-rep --page details --csv > $O/k1v2_deep_ncu_details.csv 2>/dev/null
ncu -i /tmp/k1v2_deep.ncu-rep --page raw --csv > $O/k1v2_deep_ncu_raw.csv 2>/dev/null
ncu -i /tmp/k1v2_deep.ncu-rep --page source --csv > /tmp/k1v2_src.csv 2>/dev/null
python tools/sass_lines.py paper_2412_20509_b200/libgmf_asgd.so _ZN3gmf7k_grad2ILi1ELi12EEEvNS_6ParamsExxd /tmp/k1v2_src.csv 40 --file gmf_tc2.cuh > $O/k1v2_deep_lines.txt 2>&1
ls -la $O | head -40
echo evidence done
