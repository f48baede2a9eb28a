cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/mm
./tools/micro/mulmod_rate > gpurun_out/mm/mulmod_rate.jsonl 2>&1
cat gpurun_out/mm/mulmod_rate.jsonl
