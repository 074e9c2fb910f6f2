cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/exp1.log; : > $out
for n in 4000 20000 100000; do python scripts/prof_estep.py --n $n >> $out 2>&1; done
python scripts/prof_estep.py --n 4000 --full-slice >> $out 2>&1
python scripts/prof_estep.py --n 20000 --full-slice --em-iters 3 >> $out 2>&1
for v in np1 np4; do CFUST_LIB=$PWD/paper_2005_06848_b200/libcfust_$v.so python scripts/prof_estep.py --n 20000 >> $out 2>&1; done
