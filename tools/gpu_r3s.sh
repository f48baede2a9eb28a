# experiment: later 8-stage passes with two groups (two twiddle sets) per CTA for any plan (NTT_LATER_SEP=1) vs the product
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3s}; mkdir -p $O
for i in 1 2; do
for L in libntt128.so libntt128_sep.so; do
AB_SIZES=14,16,17 NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
