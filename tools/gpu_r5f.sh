# vec128_mul's pseudo-Mersenne product (OP_MULP): BLAS parity, A/B against the previous build
# (libntt128_psmv3.so: Barrett), then the full evidence run on the product library (tools/gpu_r3t.sh)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r5f}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_vec.py -q -x > $O/pytest_vec.log 2>&1; echo "pytest vec rc=$?"; tail -3 $O/pytest_vec.log
for i in 1 2; do
for L in libntt128.so libntt128_psmv3.so; do
TAG=$L NTT128_LIB=paper_2509_12494_b200/$L timeout 300 python tools/exp_vec_graph.py >> $O/vec_ab.txt 2>&1; echo "vec $L rc=$?"
done; done
cat $O/vec_ab.txt
TAG=${TAG:-r5f} bash tools/gpu_r3t.sh
