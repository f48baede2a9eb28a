cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t8
timeout 900 python -m pytest tests/test_gpu_ntt.py -x -q -p no:cacheprovider > gpurun_out/t8/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t8/pytest_gpu.log
tail -2 gpurun_out/t8/pytest_gpu.log
for v in default rb3; do
  if [ $v = rb3 ]; then export NTT128_LIB=$PWD/paper_2509_12494_b200/libntt128_rb3.so; fi
  python bench.py --steps 10 --warmup 3 --no-rows --no-cpu-baseline > gpurun_out/t8/bench_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/t8/bench_$v.json'));print('$v', d['value'], d['roofline']['frac'], d['fwd_ms'], d['inv_ms'])"
done
