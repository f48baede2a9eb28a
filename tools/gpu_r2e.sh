# round 2: chain tests, BLAS tests + sweep check, bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_vec.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
for i in 1 2 3; do TAG="product r$i" timeout 120 python tools/exp_vec_graph.py >> $O/vec.txt 2>&1; done; cat $O/vec.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; head -c 2500 $O/bench.json; echo; python -c "
import json; d=json.load(open('$O/bench.json')); r=d['rows']; print({k: v for k, v in r.items() if 'cfg2' in k or 'polymul' in k})"
