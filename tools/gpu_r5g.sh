# ncu --set full of vec128_mul's pseudo-Mersenne kernel (k_vec<5, 2>) and axpy (k_vec<3, 1>) on the final tree
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r5g}; mkdir -p $O
python tools/exp_vec_graph.py > $O/plain.log 2>&1 && timeout 600 ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_vec<\(int\)[35]" -s 2 -c 4 -o /tmp/prof_vec python tools/exp_vec_graph.py > $O/ncu_vec.log 2>&1; echo "ncu vec rc=$?"
ncu -i /tmp/prof_vec.ncu-rep --page raw --csv > $O/prof_vec_raw.csv 2>&1
cat $O/plain.log
