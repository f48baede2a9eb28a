# round 2: TMA layout probe (pitch hypothesis); BLAS grid / unroll sweep (experiment builds)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -cudart shared -O2 -o /tmp/tma_layout tools/probe/tma_layout.cu && timeout 60 /tmp/tma_layout > $O/probe.log 2>&1; echo "probe rc=$?"; cat $O/probe.log
for u in 2 4 8; do
  for c in 3 4 5 6 8 12 16; do
    TAG="u$u ctas/sm=$c" NTT128_VEC_CTAS_PER_SM=$c NTT128_LIB=paper_2509_12494_b200/libntt128_vu$u.so timeout 120 python tools/exp_vec_graph.py >> $O/vec.txt 2>&1
  done
done
TAG="product" timeout 120 python tools/exp_vec_graph.py >> $O/vec.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_overlap.py tests/test_gpu_bitrev.py tests/test_gpu_large.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
cat $O/vec.txt
