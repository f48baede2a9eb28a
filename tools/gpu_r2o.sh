# round 2: shared-memory carveout and 17/18 CTAs per SM for the radix-4 multi-pass kernels (A/B)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2o; mkdir -p $O
for i in 1 2; do
for L in libntt128.so libntt128_co.so libntt128_o1088.so libntt128_o1152.so; do
AB_SIZES=12,13,14,16,17 NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
