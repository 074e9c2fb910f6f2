# r02 call b: cfg2 golden chunk (background) + GPU tests on the new kernel + A/B timing of kernel variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/gold
cp tests/golden/fit_cfg2_full.partial.json gpurun_out/gold/ 2>/dev/null
(python scripts/make_fit_goldens.py cfg2_full --dir gpurun_out/gold --budget-s ${GOLD_BUDGET:-1500} --threads 12 > gpurun_out/gold/cfg2.log 2>&1) &
GP=$!
python -m paper_2005_06848_b200.build > gpurun_out/build.log 2>&1
for v in old new mbq3_1; do
  lib=paper_2005_06848_b200/libcfust_$v.so; [ $v = new ] && lib=paper_2005_06848_b200/libcfust.so
  CFUST_LIB=$PWD/$lib timeout 600 python scripts/bench_configs.py --configs 1,2,3 --iters 3 > gpurun_out/ab_$v.log 2>&1
  CFUST_LIB=$PWD/$lib timeout 600 python scripts/bench_configs.py --configs 5 --scale 0.2 --iters 2 >> gpurun_out/ab_$v.log 2>&1
  CFUST_LIB=$PWD/$lib timeout 600 python scripts/bench_configs.py --configs 4 --scale 0.05 --iters 2 >> gpurun_out/ab_$v.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
wait $GP
echo "gold exit $?" >> gpurun_out/gold/cfg2.log
