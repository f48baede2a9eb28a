# round 2 final evidence (re-entry): smoke, default bench, reference arm, ncu launch list + full captures
# (cfg3 pass kernels, cfg5 four-step passes, natural-layout copy kernels), full GPU test suite
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-r3f}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi.csv 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-rows --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
$CMD > $O/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ntt_pass -s 4 -c 4 -o /tmp/prof $CMD > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/prof.ncu-rep --page raw --csv > $O/prof_raw.csv 2>&1
ncu -i /tmp/prof.ncu-rep --page details --csv > $O/prof_details.csv 2>&1
python tools/exp_fourstep_prof.py > $O/fs_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ntt_pass -s 6 -c 6 -o /tmp/prof_fs python tools/exp_fourstep_prof.py > $O/ncu_fs.log 2>&1; echo "ncu fs rc=$?"
ncu -i /tmp/prof_fs.ncu-rep --page raw --csv > $O/prof_fs_raw.csv 2>&1
python tools/exp_fourstep_nat_prof.py > $O/fsn_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none -k regex:k_fs_ -s 8 -c 4 -o /tmp/prof_fsn python tools/exp_fourstep_nat_prof.py > $O/ncu_fsn.log 2>&1; echo "ncu fsn rc=$?"
ncu -i /tmp/prof_fsn.ncu-rep --page raw --csv > $O/prof_fsn_raw.csv 2>&1
ls -la $O; du -sh $O
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest_gpu.log
