# r02 call p: chi nodes over w-sorted lattice points, SPLIT-mode prefetch of chi/W: tests + iteration times
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/iter_time.py --configs 1,3 > gpurun_out/r02p_iter_time.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_split.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fit_control.py tests/test_gpu_special.py -q -x > gpurun_out/r02p_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02p_tests.log
timeout 600 python scripts/bench_configs.py --configs 1,2 --scale 0.002 --iters 5 > gpurun_out/r02p_small.log 2>&1
