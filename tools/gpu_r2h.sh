# round 2: does a uniform (kernel-parameter) modulus raise the register-only butterfly rate?
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2h; mkdir -p $O
bash tools/micro/build.sh bfly_uniform && for i in 1 2; do ./tools/micro/bfly_uniform >> $O/bfly_uniform.jsonl 2>&1; done; cat $O/bfly_uniform.jsonl
