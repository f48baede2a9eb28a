cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pm
./tools/micro/pipe_mix2 > gpurun_out/pm/pipe_mix2.jsonl 2>&1
cat gpurun_out/pm/pipe_mix2.jsonl
