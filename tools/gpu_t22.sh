cd $GRAFT_REPO_ROOT
for v in default s10 s9; do
  if [ $v != default ]; then export NTT128_LIB=$PWD/paper_2509_12494_b200/libntt128_$v.so; else unset NTT128_LIB; fi
  echo "== $v"; python tools/exp_sizes.py 10,11,12,13
done
