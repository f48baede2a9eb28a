# later passes of one-modulus plans with group g of two polynomials per CTA (k_ntt_later_tl): parity + A/B vs NTT_LATER_TILES=1
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3r}; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_chain.py tests/test_gpu_overlap.py tests/test_gpu_large.py tests/test_capi_c.py -m gpu -q -x -k "not cfg5 and not cyclic_large and not polymul_all" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for i in 1 2; do
for L in libntt128.so libntt128_prev.so; do
AB_SIZES=13,14,16,17 NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
