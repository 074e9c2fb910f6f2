# r02 call l: q = 0 operands in the constant bank (lease holder) vs shared memory (CFUST_NO_TCONST=1)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "3- or 3] or q0 or lease or predict or shard" > gpurun_out/r02l_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02l_tests.log
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -q -x -k "3 or q0 or t_" >> gpurun_out/r02l_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02l_tests.log
for r in 1 2 3; do
  python scripts/bench_configs.py --configs 3 --iters 5 2>&1 | tail -1 | sed 's/^/tconst /' >> gpurun_out/r02l_cfg3.log
  CFUST_NO_TCONST=1 python scripts/bench_configs.py --configs 3 --iters 5 2>&1 | tail -1 | sed 's/^/smem /' >> gpurun_out/r02l_cfg3.log
done
timeout 600 python scripts/iter_time.py --configs 3 >> gpurun_out/r02l_cfg3.log 2>&1
