# round 2: uniform modulus in one-pass kernels (nq == 1) -- parity + A/B; headline bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2j; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_vec.py tests/test_capi_c.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
for i in 1 2; do
for L in paper_2509_12494_b200/libntt128.so paper_2509_12494_b200/libntt128_prev.so; do
AB_SIZES=10,11,12 NTT128_LIB=$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
timeout 900 python bench.py --no-cpu-baseline --no-cfg5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('$O/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac']); r=d['rows']; print({k: v for k, v in r.items() if 'frac' in k or 'us' in k or 'polymul_ms' in k})"
