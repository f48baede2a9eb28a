cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t2
python tools/probe/capture_api.py > gpurun_out/t2/probe.log 2>&1; cat gpurun_out/t2/probe.log
timeout 1200 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_large.py tests/test_gpu_overlap.py -m gpu -q -x > gpurun_out/t2/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/t2/pytest.log
python tools/exp_fourstep.py > gpurun_out/t2/fs.log 2>&1; cat gpurun_out/t2/fs.log
