O=gpurun_out/ev_s7; mkdir -p $O
python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
python tools/sweep_c5.py --only-d 50 --only-m 500 --only-dtype f32 > $O/c5_d50.jsonl 2>/dev/null; grep '"nstar": 65536' $O/c5_d50.jsonl | cut -c1-260
python tools/sweep_c5.py --only-d 15 --only-m 500 --only-dtype f64 --only-format dense > $O/c5_f64.jsonl 2>/dev/null; grep '"nstar": 65536' $O/c5_f64.jsonl | cut -c1-260
