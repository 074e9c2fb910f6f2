# r02 call o: split derive (matrices overlap the nu root), own lgamma, register Cholesky: full GPU suite, stamps, iteration times
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CFUST_LIB=paper_2005_06848_b200/libcfust_mprof.so timeout 300 python scripts/mprof_run.py > gpurun_out/r02o_mprof.log 2>&1
timeout 600 python scripts/iter_time.py --configs 1,3 > gpurun_out/r02o_iter_time.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r02o_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02o_pytest_gpu.log
