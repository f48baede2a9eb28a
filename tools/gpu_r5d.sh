# pseudo-Mersenne class v2 (product < Q, single-fold add / sub): A/B against the v1 build
# (double folds, libntt128_psmv1.so) and the no-PSM build, then the full evidence run (tools/gpu_r3t.sh)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r5d}; mkdir -p $O
for i in 1 2; do
for L in libntt128.so libntt128_psmv1.so libntt128_nopsm.so; do
AB_SIZES=12,14,16,17 NTT128_LIB=paper_2509_12494_b200/$L timeout 600 python tools/exp_ab.py >> $O/ab.txt 2>&1; echo "ab $L rc=$?"
done; done
cat $O/ab.txt
TAG=${TAG:-r5d} bash tools/gpu_r3t.sh
