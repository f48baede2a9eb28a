# 6-word (192-bit) NTT: register budget of the pass kernels (NTT256_MINB6 = 1 / 12 / 16 resident CTAs per SM)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3k}; mkdir -p $O
for r in 1 2; do
PRIME=b256 timeout 300 python tools/exp_ntt256.py 12,16,18 >> $O/ab.txt 2>&1
for L in libntt128.so libntt128_m6_12.so libntt128_m6_16.so; do
echo "== $L" >> $O/ab.txt
PRIME=b192 NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ntt256.py 12,16,18 >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
