cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t9
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t9/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t9/pytest_gpu.log
tail -2 gpurun_out/t9/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/t9/bench.json 2> gpurun_out/t9/bench.err; echo "bench rc=$?"
cat gpurun_out/t9/bench.json
timeout 900 bash tools/gpu_prof.sh t9p
python tools/ncu_summary.py gpurun_out/t9p/prof.ncu-rep 2 > gpurun_out/t9p/summary.txt 2>&1
ncu -i gpurun_out/t9p/prof.ncu-rep --page source --csv --print-source sass > gpurun_out/t9p/source.csv 2>/dev/null
