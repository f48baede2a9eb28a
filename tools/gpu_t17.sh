cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t17
for v in default c2 c1; do
  if [ $v != default ]; then export NTT128_LIB=$PWD/paper_2509_12494_b200/libntt128_$v.so; else unset NTT128_LIB; fi
  python bench.py --steps 20 --warmup 5 --no-rows --no-cpu-baseline > gpurun_out/t17/bench_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/t17/bench_$v.json'));print('$v', '%.4e'%d['value'], d['roofline']['frac'], '%.4f %.4f'%(d['fwd_ms'], d['inv_ms']))"
done
