cd $GRAFT_REPO_ROOT
O=gpurun_out/t8; mkdir -p $O
python tools/exp_fourstep.py > $O/fs.log 2>&1; cat $O/fs.log
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; head -c 3000 $O/bench.json
