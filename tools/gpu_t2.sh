cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t2
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/t2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t2/pytest_gpu.log
tail -40 gpurun_out/t2/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/t2/bench.json 2> gpurun_out/t2/bench.err; echo "bench rc=$?"
cat gpurun_out/t2/bench.json; tail -20 gpurun_out/t2/bench.err
