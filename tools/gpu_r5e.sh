# pseudo-Mersenne class v3 (fold constants selected on the carry predicate): A/B against the v2 build
# (libntt128_psmv2.so), then the full evidence run on the product library (tools/gpu_r3t.sh)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r5e}; mkdir -p $O
for i in 1 2; do
for L in libntt128.so libntt128_psmv2.so; do
AB_SIZES=12,14,16,17 NTT128_LIB=paper_2509_12494_b200/$L timeout 600 python tools/exp_ab.py >> $O/ab.txt 2>&1; echo "ab $L rc=$?"
done; done
cat $O/ab.txt
TAG=${TAG:-r5e} bash tools/gpu_r3t.sh
