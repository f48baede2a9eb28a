# round 2: full GPU suite with chain + shift scaling; A/B of N^-1 by shifting
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2f; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -12 $O/pytest_gpu.log
for i in 1 2; do
for L in paper_2509_12494_b200/libntt128.so paper_2509_12494_b200/libntt128_noshift.so; do
AB_SIZES=12,16,17 NTT128_LIB=$L timeout 300 python tools/exp_ab.py >> $O/ab.txt 2>&1
done; done
cat $O/ab.txt
