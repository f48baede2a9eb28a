# usage: bash tools/gpu_variants.sh "name1 name2 ..."  -- headline bench with each experimental library build
cd $GRAFT_REPO_ROOT
for v in default $1; do
  if [ $v != default ]; then export NTT128_LIB=$PWD/paper_2509_12494_b200/libntt128_$v.so; else unset NTT128_LIB; fi
  python bench.py --no-rows --no-cpu-baseline --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4e'%d['value'], d['roofline']['frac'], d['fwd_ms'], d['inv_ms'])"
done
