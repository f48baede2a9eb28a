cd $GRAFT_REPO_ROOT
O=gpurun_out/t5; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_vec.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.log
python tools/exp_fourstep.py > $O/fs.log 2>&1; cat $O/fs.log
for c in 0 1 2; do for m in 0 28; do TAG="cfg$c pipe$m" NTT128_VEC_PIPE_CFG=$c NTT128_VEC_PIPE=$m NTT128_LIB=$PWD/paper_2509_12494_b200/libntt128_exp.so python tools/exp_vec_graph.py; done; done > $O/vec.log 2>&1; cat $O/vec.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fs_launches.csv python tools/exp_fourstep_prof.py > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py $O/fs_launches.csv 2>&1 | grep k_ntt
