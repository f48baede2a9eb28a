# BLAS: software-prefetch grid-stride kernel (experiment build) vs the product shape, cfg2 graph replays
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3d}; mkdir -p $O
L=paper_2509_12494_b200/libntt128_exp.so
for r in 1 2; do
  TAG="product r$r" timeout 120 python tools/exp_vec_graph.py >> $O/vec.txt 2>&1
  for d in 1 2 3; do for c in 4 6 8 12 16; do
    TAG="pf D=$d ctas/sm=$c r$r" NTT128_VEC_PF=$d NTT128_VEC_PF_CTAS=$c NTT128_LIB=$L timeout 120 python tools/exp_vec_graph.py >> $O/vec.txt 2>&1
  done; done
done
cat $O/vec.txt
