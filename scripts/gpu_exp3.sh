cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/exp3.log; : > $out
for v in default ew8m2h ew4m4 ew4m5 ew4m6 ew8m3; do
  if [[ $v == default ]]; then L=$PWD/paper_2005_06848_b200/libcfust.so; else L=$PWD/paper_2005_06848_b200/libcfust_$v.so; fi
  for n in 20000 100000; do CFUST_LIB=$L python scripts/prof_estep.py --n $n --reps 2 >> $out 2>&1; done
  CFUST_LIB=$L python scripts/prof_estep.py --config 4 --n 2000 --reps 1 >> $out 2>&1
  CFUST_LIB=$L python scripts/prof_estep.py --config 5 --n 200000 --reps 1 >> $out 2>&1
done
