cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t10
timeout 1200 python -m pytest tests/test_gpu_fourstep.py -x -q -p no:cacheprovider --durations=5 > gpurun_out/t10/pytest_fs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t10/pytest_fs.log
tail -12 gpurun_out/t10/pytest_fs.log
