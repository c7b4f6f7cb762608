#!/bin/bash
# build an alternative library from a csrc copy: tools/build_alt.sh alt/w8  -> alt/w8/libgmf_asgd.so (A/B via GMF_LIB_PATH)
set -e
D="$1"; mkdir -p "$D/_build"
pids=()
for f in "$D"/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I /root/repo/include -I "$D/csrc" -c "$f" -o "$D/_build/$(basename $f).o" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared --cudart static -o "$D/libgmf_asgd.so" "$D"/_build/*.o
ls -la "$D/libgmf_asgd.so"
