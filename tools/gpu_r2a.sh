# round 2: TMA tile loads of later passes -- parity, A/B against the cp.async build
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_overlap.py tests/test_gpu_fourstep.py tests/test_gpu_bitrev.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for i in 1 2; do
for L in paper_2509_12494_b200/libntt128.so paper_2509_12494_b200/libntt128_notma.so; do
AB_SIZES=12,13,14,15,16,17 NTT128_LIB=$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
