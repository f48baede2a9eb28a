# round 2: chained calls (tests + A/B); BLAS sweep part 2 (smaller tiles, more waves)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_chain.py -m gpu -q -x > $O/pytest_chain.log 2>&1; echo "pytest chain rc=$?"; tail -15 $O/pytest_chain.log
timeout 600 python tools/exp_chain.py > $O/chain_ab.txt 2>&1; echo "chain ab rc=$?"; cat $O/chain_ab.txt
for L in vu2 vu1t256 vu2t128 vu1t128; do
  for c in 16 24 32 64; do
    TAG="$L ctas/sm=$c" NTT128_VEC_CTAS_PER_SM=$c NTT128_LIB=paper_2509_12494_b200/libntt128_$L.so timeout 120 python tools/exp_vec_graph.py >> $O/vec.txt 2>&1
  done
done
cat $O/vec.txt
