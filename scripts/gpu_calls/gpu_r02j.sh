# r02 call j: q = 0 kernel with TMA-staged y tiles (cur) vs the L1-load version (notma) and an exp-table build
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -q -x -k "3 or q0 or t_" > gpurun_out/r02j_q0_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02j_q0_tests.log
bash scripts/gpu_calls/gpu_cfg3.sh cur notma exptab
