# round 2: 256-bit uniform modulus + shift scaling (parity, A/B); register-budget / radix variants of the 8/9-stage kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ntt256.py -m gpu -q -x > $O/pytest256.log 2>&1; echo "pytest256 rc=$?"; tail -3 $O/pytest256.log
for i in 1 2; do for L in libntt128.so libntt128_prev.so; do NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ntt256.py > $O/n256_$L.$i.txt 2>&1; echo "$L: $(tail -3 $O/n256_$L.$i.txt | tr '\n' ' ')"; done; done
for i in 1 2; do
for L in libntt128.so libntt128_rb8_3.so libntt128_occ1024.so libntt128_rb8_3_occ1024.so; do
AB_SIZES=12,14,15,16,17 NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
