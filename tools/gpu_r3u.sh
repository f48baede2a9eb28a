# experiment: 9-stage first passes with two tiles per CTA and radix-4 rounds (128 threads, 64 registers) vs the product
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3u}; mkdir -p $O
for i in 1 2; do
for L in libntt128.so libntt128_f9r2.so; do
AB_SIZES=15,17 NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
