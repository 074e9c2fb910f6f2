# r02 call s: q = 0 E-step with table-driven log1p / exp in shared memory (cur) vs polynomial (notab)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "3 or q0 or t_ or predict" > gpurun_out/r02s_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02s_tests.log
bash scripts/gpu_calls/gpu_cfg3.sh cur notab
