# usage: bash tools/store_evidence.sh <tag> -- copy gpurun_out/<tag> (tools/gpu_r3t.sh output) into profiles/r02/final
set -e
T=$1; S=gpurun_out/$T; D=profiles/r02/final
cp $S/bench.json $S/bench_ref.json $S/smoke.log $S/sanitize_driver.log $S/launches.csv $S/prof_raw.csv $S/smi.csv $D/
python tools/launch_summary.py $S/launches.csv > $D/launch_summary.txt
python tools/ncu_summary.py $S/prof_raw.csv > $D/ncu_full_summary.txt
python tools/ncu_traffic.py $S/prof_raw.csv profiles/ncu_traffic.json "profiles/r02/final (ncu --set full -k regex:k_ntt -s 4 -c 4, bench.py --steps 2 --warmup 3 --no-rows --no-cpu-baseline; final kernels: k_ntt_first_tl first passes, k_ntt_pass later passes, pseudo-Mersenne class)" > /dev/null
tail -12 $S/pytest_gpu.log > profiles/r02/pytest_gpu_final_tail.txt
