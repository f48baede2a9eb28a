cd $GRAFT_REPO_ROOT
O=gpurun_out/t7; mkdir -p $O
L=$PWD/paper_2509_12494_b200
for i in 1 2; do
python tools/exp_ab.py 2>&1 | tail -1
NTT128_LIB=$L/libntt128_bulk1.so python tools/exp_ab.py 2>&1 | tail -1
NTT128_LIB=$L/libntt128_bulk2.so python tools/exp_ab.py 2>&1 | tail -1
done > $O/ab.log; cat $O/ab.log
python tools/exp_fourstep.py > $O/fs.log 2>&1; NTT128_LIB=$L/libntt128_fsc8.so python tools/exp_fourstep.py >> $O/fs.log 2>&1; cat $O/fs.log
