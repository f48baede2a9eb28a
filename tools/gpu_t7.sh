cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t7
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t7/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t7/pytest_gpu.log
tail -3 gpurun_out/t7/pytest_gpu.log
timeout 900 bash tools/gpu_prof.sh t7p
python tools/ncu_summary.py gpurun_out/t7p/prof.ncu-rep 2 > gpurun_out/t7p/summary.txt 2>&1
cat gpurun_out/t7p/plain.json | cut -c1-300
