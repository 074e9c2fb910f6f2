# usage: bash scripts/gpu_calls/gpu_variants.sh lib1 lib2 ...   (names of paper_2005_06848_b200/libcfust_<name>.so)
# E-step timing of experiment builds on cfg2 / cfg5 / cfg4 slices -> gpurun_out/variants.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "$@"; do
  for spec in "2 20000" "5 200000" "4 2000" "1 200000"; do
    set -- $spec
    CFUST_LIB=paper_2005_06848_b200/libcfust_$v.so timeout 300 python scripts/prof_estep.py --config $1 --n $2 --reps 2 >> gpurun_out/variants.log 2>&1
  done
done
