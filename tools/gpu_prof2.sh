# usage: bash tools/gpu_prof2.sh <tag>  -- ncu --set full of the two cfg3 pass kernels (+ source page) and the register-only butterfly kernel
cd $GRAFT_REPO_ROOT
T=${1:-p}
O=gpurun_out/$T
mkdir -p $O
CMD="python bench.py --steps 2 --warmup 3 --no-rows --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ntt_pass -s 4 -c 2 -o $O/prof $CMD > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bfly -s 3 -c 1 -o $O/prof_bfly ./tools/micro/bfly_rate > $O/ncu_bfly.log 2>&1; echo "ncu bfly rc=$?"
