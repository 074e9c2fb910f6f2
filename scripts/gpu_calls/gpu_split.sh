# Small-n E-step: warps per observation forced to 1/2/4/8 (CFUST_SPLIT) and automatic (0),
# cfg1/cfg2/cfg5/cfg4 shapes at AIS size (n = 202) and up -> gpurun_out/split.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for spec in "1 202" "1 1000" "1 3000" "2 202" "2 1000" "2 3000" "5 1000" "5 3000" "4 202" "4 1000"; do
  set -- $spec
  for sp in 1 2 4 8 0; do
    CFUST_SPLIT=$sp timeout 300 python scripts/prof_estep.py --config $1 --n $2 --reps 5 2>&1 | sed "s/^/split=$sp /" >> gpurun_out/split.log
  done
done
