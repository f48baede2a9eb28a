cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t4
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t4/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t4/pytest_gpu.log
tail -5 gpurun_out/t4/pytest_gpu.log
timeout 900 bash tools/gpu_prof.sh t4p
cat gpurun_out/t4p/plain.json
