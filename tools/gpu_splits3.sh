# usage: bash tools/gpu_splits3.sh -- three-pass split candidates (NTT128_SPLIT experiment switch)
cd $GRAFT_REPO_ROOT
for c in 19: 19:5,6,8 19:6,5,8 19:5,8,6 20: 20:6,6,8 20:5,7,8 20:6,8,6 20:9,5,6 21: 21:5,8,8 21:8,5,8 21:9,6,6 21:6,6,9 22: 22:6,8,8 22:8,6,8 22:9,5,8 23: 23:7,8,8 23:9,6,8 23:6,9,8 23:9,9,5; do
  n=${c%%:*}; sp=${c#*:}
  r=$(NTT128_SPLIT=$sp python tools/exp_sizes.py $n | tail -1)
  echo "[$sp] -> $r"
done
