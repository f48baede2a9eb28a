# usage: bash tools/gpu_tests.sh <tag> [pytest args] -- full GPU suite (no -x), durations, then a short bench
cd $GRAFT_REPO_ROOT
T=${1:-t}; shift
O=gpurun_out/$T
mkdir -p $O
nproc > $O/host.txt; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> $O/host.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=25 ${@} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest_gpu.log; tail -40 $O/pytest_gpu.log
timeout 300 python bench.py --no-rows --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json | head -c 1500
