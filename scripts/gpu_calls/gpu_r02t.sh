# r02 call t: C11 calibrated monotonicity on the full cfg2 fit, and the default bench (cfg5)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CFUST_MONOTONE_REPORT=gpurun_out/r02t_monotone_cfg2.json timeout 900 python -m pytest tests/test_gpu_monotone.py -q -s > gpurun_out/r02t_monotone.log 2>&1; echo "exit $?" >> gpurun_out/r02t_monotone.log
timeout 1200 python bench.py > gpurun_out/r02t_bench.log 2> gpurun_out/r02t_bench.err; echo "bench exit $?" >> gpurun_out/r02t_bench.err
