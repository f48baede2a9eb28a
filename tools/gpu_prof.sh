# usage: bash tools/gpu_prof.sh <tag>  -- plain bench, ncu launch list, ncu --set full of k_ntt_pass
cd $GRAFT_REPO_ROOT
T=${1:-p}
O=gpurun_out/$T
mkdir -p $O
CMD="python bench.py --steps 2 --warmup 3 --no-rows --no-cpu-baseline"
$CMD > $O/plain.json 2> $O/plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ntt_pass -s 4 -c 2 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "rc=$?"
tail -3 $O/ncu_full.log
