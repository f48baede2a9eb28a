# usage: bash tools/gpu_quick.sh <tag> [extra command]  -- gpu tests + bench (no rows) + optional extra
cd $GRAFT_REPO_ROOT
T=${1:-q}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 300 python bench.py --no-rows --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json
if [ -n "$2" ]; then bash -c "$2" > $O/extra.log 2>&1; echo "extra rc=$?"; cat $O/extra.log | tail -30; fi
