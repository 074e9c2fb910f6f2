# r02 call k: phase-2 rework (w rows in shared memory, S2 by one DMMA) with / without TMA-staged y, vs the old kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -q -x -k "3 or q0 or t_" > gpurun_out/r02k_q0_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02k_q0_tests.log
rm -f gpurun_out/cfg3.log
bash scripts/gpu_calls/gpu_cfg3.sh cur p2notma notma
