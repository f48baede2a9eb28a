cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t3
timeout 300 python -m pytest tests/test_gpu_vec.py -q -p no:cacheprovider > gpurun_out/t3/pytest_vec.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t3/pytest_vec.log
tail -3 gpurun_out/t3/pytest_vec.log
timeout 900 bash tools/gpu_prof.sh t3p
