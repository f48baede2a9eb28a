# final tree (two-tile first / later passes): smoke, bench, reference arm, self-checking driver,
# ncu launch list + full capture of the cfg3 passes, full GPU test suite
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3t}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi.csv 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 300 python tools/sanitize_driver.py > $O/sanitize_driver.log 2>&1; echo "driver rc=$?"; tail -1 $O/sanitize_driver.log
CMD="python bench.py --steps 2 --warmup 3 --no-rows --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
$CMD > $O/plain2.log 2>&1 && timeout 900 ncu -f --set full --clock-control none --import-source on -k "regex:k_ntt" -s 4 -c 4 -o /tmp/prof $CMD > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/prof.ncu-rep --page raw --csv > $O/prof_raw.csv 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest_gpu.log
