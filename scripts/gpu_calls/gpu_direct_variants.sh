# E-step timing of the SOV-direct estimator for experiment builds: bash scripts/gpu_calls/gpu_direct_variants.sh lib...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" >> gpurun_out/dvariants.log
  CFUST_LIB=paper_2005_06848_b200/libcfust_$v.so python scripts/bench_configs.py --estimator direct --configs 1,2,4,5 --scale 0.05 --iters 2 >> gpurun_out/dvariants.log 2>&1
done
