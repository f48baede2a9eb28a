cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/t1/smi.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/t1/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/t1/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t1/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t1/pytest_gpu.log
tail -30 gpurun_out/t1/pytest_gpu.log
cat gpurun_out/t1/smoke.log
