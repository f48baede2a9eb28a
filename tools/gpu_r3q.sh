# 9-stage first passes with two groups per CTA (NTT_FIRST_TILES9=2) vs one
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3q}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ntt.py -m gpu -q -x -k "two_pass or three_pass or cfg3" > $O/pytest_t9.log 2>&1 < /dev/null; echo "(product lib) pytest rc=$?"
for i in 1 2; do
for L in libntt128.so libntt128_t9.so; do
AB_SIZES=15,16,17 NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
