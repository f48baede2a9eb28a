# lazy class of the wide-modulus kernels (q < R/4: b254 on 8 words, b190 on 6): GPU parity of the
# 256-bit suite, then A/B against a build with NTT256_LAZY=0 (every plan canonical)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r4b}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ntt256.py -q -x > $O/pytest_ntt256.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_ntt256.log
for i in 1 2; do
for L in libntt128.so libntt128_nolazy.so; do
for K in b254 b190 b256 b192; do
echo "lib $L" >> $O/ab.txt
PRIME=$K NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ntt256.py 12,16,20 >> $O/ab.txt 2>&1
done; done; done
cat $O/ab.txt
