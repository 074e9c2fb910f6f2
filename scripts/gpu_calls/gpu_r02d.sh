# r02 call d: A/B of the paired-integral loop variants + GPU tests (new parity harness) + golden chunk
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/gold
if [ -f tests/golden/fit_cfg2_full.partial.json ]; then
  cp tests/golden/fit_cfg2_full.partial.json gpurun_out/gold/
  (python scripts/make_fit_goldens.py cfg2_full --dir gpurun_out/gold --budget-s ${GOLD_BUDGET:-1500} --threads 12 > gpurun_out/gold/cfg2.log 2>&1) &
  GP=$!
fi
python -m paper_2005_06848_b200.build > gpurun_out/build.log 2>&1
for v in ${VARIANTS:-old new np1 q3np2 q3np2mb1}; do
  lib=paper_2005_06848_b200/libcfust_$v.so; [ $v = new ] && lib=paper_2005_06848_b200/libcfust.so
  CFUST_LIB=$PWD/$lib timeout 600 python scripts/bench_configs.py --configs 2 --iters 2 > gpurun_out/ab_$v.log 2>&1
  CFUST_LIB=$PWD/$lib timeout 600 python scripts/bench_configs.py --configs 5 --scale 0.2 --iters 2 >> gpurun_out/ab_$v.log 2>&1
  CFUST_LIB=$PWD/$lib timeout 600 python scripts/bench_configs.py --configs 4 --scale 0.05 --iters 2 >> gpurun_out/ab_$v.log 2>&1
done
if [ -z "$NOTEST" ]; then
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
if [ -n "$GP" ]; then wait $GP; echo "gold exit $?" >> gpurun_out/gold/cfg2.log; fi
