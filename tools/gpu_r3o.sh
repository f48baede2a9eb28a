# first pass with two groups per CTA (k_ntt_first_tl): parity on the core GPU suites + A/B vs NTT_FIRST_TILES=1
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3o}; mkdir -p $O
#timeout 1800 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_chain.py tests/test_gpu_overlap.py tests/test_capi_c.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for i in 1 2 3; do
for L in paper_2509_12494_b200/libntt128.so paper_2509_12494_b200/libntt128_prev.so; do
AB_SIZES=16 NTT128_LIB=$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
