# first pass, groups per CTA: TL = 1 (prev) / 2 (product) / 3 / 4
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3p}; mkdir -p $O
for i in 1 2; do
for L in libntt128.so libntt128_prev.so libntt128_tl3.so libntt128_tl4.so; do
AB_SIZES=16 NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
