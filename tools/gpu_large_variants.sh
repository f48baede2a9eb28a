# usage: bash tools/gpu_large_variants.sh "name1 name2" "20,23,26"  -- large-N sweep with experimental builds
cd $GRAFT_REPO_ROOT
for v in default $1; do
  if [ $v != default ]; then export NTT128_LIB=$PWD/paper_2509_12494_b200/libntt128_$v.so; else unset NTT128_LIB; fi
  echo "== $v"; python tools/exp_large.py $2
done
