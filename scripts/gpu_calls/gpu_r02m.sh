# r02 call m: M-step critical path (clock64 stamps per warp, CFUST_MSTEP_PROF build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CFUST_LIB=paper_2005_06848_b200/libcfust_mprof.so timeout 300 python scripts/mprof_run.py > gpurun_out/r02m_mprof.log 2>&1
