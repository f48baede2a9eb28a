cd $GRAFT_REPO_ROOT
O=gpurun_out/r2l; mkdir -p $O
for i in 1 2; do for L in libntt128.so libntt128_prev.so; do echo "== $L" >> $O/n256.txt; NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ntt256.py 10,12,14,16,18 >> $O/n256.txt 2>&1; done; done
cat $O/n256.txt
