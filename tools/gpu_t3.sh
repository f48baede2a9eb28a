cd $GRAFT_REPO_ROOT
O=gpurun_out/t3; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fourstep.py tests/test_gpu_overlap.py tests/test_gpu_large.py -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -8 $O/pytest.log
python tools/exp_fourstep.py > $O/fs.log 2>&1; cat $O/fs.log
python tools/micro/int_peak.py > $O/int_peak.log 2>&1; echo "int_peak rc=$?"; cp profiles/int_peak.json $O/ 2>/dev/null; grep -E "products_per_clk|ops_per_clk_per_sm_nvml|sm_mhz_median" $O/int_peak.log | head -20
