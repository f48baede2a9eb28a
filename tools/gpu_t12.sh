cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t12
timeout 900 python -m pytest tests/test_gpu_ntt.py -x -q -p no:cacheprovider > gpurun_out/t12/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t12/pytest.log
tail -2 gpurun_out/t12/pytest.log
timeout 900 bash tools/gpu_prof.sh t12p
python tools/ncu_summary.py gpurun_out/t12p/prof.ncu-rep 2 > gpurun_out/t12p/summary.txt 2>&1
ncu -i gpurun_out/t12p/prof.ncu-rep --page source --csv --print-source sass > gpurun_out/t12p/source.csv 2>/dev/null
cat gpurun_out/t12p/summary.txt; cat gpurun_out/t12p/plain.json | cut -c1-200
