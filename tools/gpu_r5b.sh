# pseudo-Mersenne class (csrc/psm128.cuh): parity first (A/B script's oracle checks, the NTT / large
# GPU tests), then A/B against a build with NTT_PSM=0 on cfg3 / cfg4 / cfg5
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r5b}; mkdir -p $O
AB_SIZES=13,14,16,17 timeout 600 python tools/exp_ab.py > $O/ab_psm.txt 2>&1; echo "ab psm rc=$?"; tail -3 $O/ab_psm.txt
AB_SIZES=13,14,16,17 NTT128_LIB=paper_2509_12494_b200/libntt128_nopsm.so timeout 600 python tools/exp_ab.py > $O/ab_nopsm.txt 2>&1; echo "ab nopsm rc=$?"; tail -1 $O/ab_nopsm.txt
timeout 1500 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_chain.py tests/test_gpu_overlap.py -q -x > $O/pytest_ntt.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_ntt.log
AB_SIZES=15 timeout 600 python tools/exp_ab.py >> $O/ab_psm.txt 2>&1
AB_SIZES=15 NTT128_LIB=paper_2509_12494_b200/libntt128_nopsm.so timeout 600 python tools/exp_ab.py >> $O/ab_nopsm.txt 2>&1
tail -1 $O/ab_psm.txt; tail -1 $O/ab_nopsm.txt
timeout 600 python tools/exp_large.py > $O/large_psm.txt 2>&1; tail -3 $O/large_psm.txt
