cd $GRAFT_REPO_ROOT
for c in 13:5,8 13:8,5 13:6,7 13:7,6 14:5,9 14:9,5 14:6,8 14:8,6 14:7,7 15:6,9 15:9,6 15:7,8 15:8,7 16:7,9 16:9,7 16:8,8 17:8,9 17:9,8 18:9,9; do
  n=${c%%:*}; sp=${c#*:}
  r=$(NTT128_SPLIT=$sp python tools/exp_sizes.py $n | tail -1)
  echo "$sp -> $r"
done
