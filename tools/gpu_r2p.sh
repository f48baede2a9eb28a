# round 2: mont_core formulation micro-benchmark (tools/micro/mont_alt.cu)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2p; mkdir -p $O
bash tools/micro/build.sh mont_alt && for i in 1 2; do ./tools/micro/mont_alt >> $O/mont_alt.jsonl 2>&1; done; cat $O/mont_alt.jsonl
