cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do
  for v in cur q3m3 q3m1; do
    lib=paper_2005_06848_b200/libcfust_$v.so; [ "$v" = cur ] && lib=paper_2005_06848_b200/libcfust.so
    CFUST_LIB=$lib timeout 600 python scripts/prof_estep.py --config 5 --n 10000000 --reps 1 2>&1 | sed "s/^/$v /" | cut -d" " -f1,3,4,8
  done
done
