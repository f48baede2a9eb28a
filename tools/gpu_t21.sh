cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t21
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t21/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t21/pytest.log
tail -2 gpurun_out/t21/pytest.log
python bench.py --steps 20 --warmup 5 --no-rows --no-cpu-baseline > gpurun_out/t21/bench.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/t21/bench.json'));print('%.4e'%d['value'], d['roofline']['frac'], '%.4f %.4f'%(d['fwd_ms'], d['inv_ms']))"
