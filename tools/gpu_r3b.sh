# natural block layout four-step: GPU parity (virtual ranks, full cfg5) and the bench row
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3b}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_large.py -k "natural or fourstep" -q -x > $O/pytest_fs.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_fs.log
timeout 600 python bench.py --steps 20 --sweep 16 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('$O/bench.json')); print({k: v for k, v in d['rows'].items() if 'cfg5' in k})"
