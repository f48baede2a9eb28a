cd $GRAFT_REPO_ROOT
timeout 900 bash tools/gpu_prof.sh t15p
python tools/ncu_summary.py gpurun_out/t15p/prof.ncu-rep 2 > gpurun_out/t15p/summary.txt 2>&1
ncu -i gpurun_out/t15p/prof.ncu-rep --page source --csv --print-source sass > gpurun_out/t15p/source.csv 2>/dev/null
cat gpurun_out/t15p/summary.txt
