cd $GRAFT_REPO_ROOT
./tools/micro/bfly_rate16 | grep variant
./tools/micro/bfly_rate | grep variant
