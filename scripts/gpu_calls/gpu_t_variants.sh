# q = 0 kernel timing for experiment builds: bash scripts/gpu_calls/gpu_t_variants.sh lib...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" >> gpurun_out/tvariants.log
  CFUST_LIB=paper_2005_06848_b200/libcfust_$v.so python scripts/bench_configs.py --configs 3 --iters 5 >> gpurun_out/tvariants.log 2>&1
done
