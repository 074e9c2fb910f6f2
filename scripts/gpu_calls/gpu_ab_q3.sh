cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2 3; do
  for spec in "5 300000" "1 100000"; do
    set -- $spec
    for v in prev cur q2n2; do
      lib=paper_2005_06848_b200/libcfust_$v.so; [ "$v" = cur ] && lib=paper_2005_06848_b200/libcfust.so
      CFUST_LIB=$lib timeout 300 python scripts/prof_estep.py --config $1 --n $2 --reps 2 2>&1 | sed "s/^/$v /" >> gpurun_out/ab2.log
    done
  done
done
