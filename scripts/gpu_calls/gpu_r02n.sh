# r02 call n: M-step latency work (warp-wide nu root with interleaved psi/psi', one-pass transcendental
# constants in derive, Sigma's factor carried from the M-step into derive): tests, stamps, iteration times
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_special.py tests/test_gpu_fit_control.py tests/test_gpu_parity.py tests/test_gpu_init.py -q -x > gpurun_out/r02n_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02n_tests.log
CFUST_LIB=paper_2005_06848_b200/libcfust_mprof.so timeout 300 python scripts/mprof_run.py > gpurun_out/r02n_mprof.log 2>&1
timeout 600 python scripts/iter_time.py --configs 1,3 > gpurun_out/r02n_iter_time.log 2>&1
