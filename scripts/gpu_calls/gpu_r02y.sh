# r02 call y (HEAD parity evidence beyond the -m gpu suite): the 1200-case wide fuzz (3 seeds x 400, every pair),
# the -m slow full 10^4-observation cfg4 subsample (protocol (i)-(ii)), and the cfg2 bench line (round 1's workload).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for seed in 777 4242 99; do
  CFUST_FUZZ_N=400 CFUST_FUZZ_SEED=$seed timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q 2>&1 | tail -1 | sed "s/^/seed $seed: /" >> gpurun_out/r02y_fuzz_wide.log
done
timeout 1500 python -m pytest tests/test_slow_fullsize.py -m slow -q > gpurun_out/r02y_pytest_slow.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02y_pytest_slow.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/r02y_bench_cfg2.log 2> gpurun_out/r02y_bench_cfg2.err; echo "bench exit $?" >> gpurun_out/r02y_bench_cfg2.err
