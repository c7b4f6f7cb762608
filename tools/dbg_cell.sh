S="python tools/sweep_c5.py --only-m 500 --only-d 15 --only-dtype f32 --only-family poisson --only-nstar 65536 --only-format csr --steps 10 --warmup 2"
echo "== main"; timeout 300 $S 2>&1 | grep -v "^{\"gen\|peak" | tail -4 | cut -c1-300
echo "== main nb"; timeout 300 python tools/sweep_c5.py --only-m 500 --only-d 15 --only-dtype f32 --only-family nb --only-nstar 65536 --only-format csr --steps 10 --warmup 2 2>&1 | grep -v "^{\"gen\|peak" | tail -3 | cut -c1-300
echo "== head"; GMF_LIB_PATH=/root/repo/alt/head/libgmf_asgd.so timeout 300 $S 2>&1 | grep -v "^{\"gen\|peak" | tail -4 | cut -c1-300
echo "== main v1"; GMF_TC_VERSION=1 timeout 300 $S 2>&1 | grep -v "^{\"gen\|peak" | tail -3 | cut -c1-300
echo "== sanitizer"; timeout 600 compute-sanitizer --tool memcheck $S 2>&1 | grep -v "^{\"gen\|peak" | head -40 | cut -c1-300
