# usage: bash scripts/gpu_calls/gpu_ab.sh libA libB ...  (paper_2005_06848_b200/libcfust_<name>.so or "cur" = libcfust.so)
# E-step ms of each build on cfg1 / cfg5 / cfg2 / cfg4 slices, interleaved, 2 rounds -> gpurun_out/ab.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do
  for spec in "1 40000" "5 100000" "2 20000" "4 2000"; do
    set -- $spec
    for v in "${@:3}" $LIBS; do :; done
    for v in $LIBS; do
      lib=paper_2005_06848_b200/libcfust_$v.so; [ "$v" = cur ] && lib=paper_2005_06848_b200/libcfust.so
      CFUST_LIB=$lib timeout 300 python scripts/prof_estep.py --config $1 --n $2 --reps 2 2>&1 | sed "s/^/$v /" >> gpurun_out/ab.log
    done
  done
done
