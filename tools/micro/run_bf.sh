cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bf
./tools/micro/bfly_rate > gpurun_out/bf/bfly_rate.jsonl 2>&1
cat gpurun_out/bf/bfly_rate.jsonl
