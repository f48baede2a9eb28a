cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t18
timeout 900 python -m pytest tests/test_gpu_ntt.py tests/test_gpu_fourstep.py -x -q -p no:cacheprovider > gpurun_out/t18/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t18/pytest.log
tail -2 gpurun_out/t18/pytest.log
for v in pipe nopipe; do
  if [ $v = nopipe ]; then export NTT128_NO_PIPE=1; else unset NTT128_NO_PIPE; fi
  python bench.py --steps 20 --warmup 5 --no-rows --no-cpu-baseline > gpurun_out/t18/bench_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/t18/bench_$v.json'));print('$v', '%.4e'%d['value'], d['roofline']['frac'], '%.4f %.4f'%(d['fwd_ms'], d['inv_ms']))"
done
