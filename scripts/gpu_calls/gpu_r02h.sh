# r02 call h: pipe/Phi microbenchmarks; A/B of the special-function variants (even/odd Horner, FP32 reciprocal seed)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 ./tools/bench_pipes > gpurun_out/bench_pipes.log 2>&1
for r in 1 2; do
  for spec in "5 2000000" "2 100000" "4 50000" "3 4000000"; do
    set -- $spec
    for v in cur eo f32 eof32; do
      lib=paper_2005_06848_b200/libcfust_$v.so; [ "$v" = cur ] && lib=paper_2005_06848_b200/libcfust.so
      CFUST_LIB=$lib timeout 300 python scripts/prof_estep.py --config $1 --n $2 --reps 2 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/ab_eo.log
    done
  done
done
