# round 2: uniform modulus in the load/store factor paths (four-step pass C, negacyclic twist/untwist, polymul point-wise) -- parity + A/B
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2m; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_fourstep.py tests/test_gpu_bitrev.py tests/test_gpu_chain.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for i in 1 2; do for L in libntt128.so libntt128_prev.so; do
  echo "== $L" >> $O/ab.txt
  NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_fourstep.py >> $O/ab.txt 2>&1
  NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_polymul.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
