cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/exp4.log; : > $out
./tools/bench_sov >> $out 2>&1; ./tools/bench_sov_lib >> $out 2>&1
for n in 100000; do python scripts/prof_estep.py --n $n --reps 2 >> $out 2>&1; done
python scripts/prof_estep.py --config 4 --n 2000 --reps 1 >> $out 2>&1
python scripts/prof_estep.py --config 5 --n 200000 --reps 1 >> $out 2>&1
timeout 1200 python -m pytest tests/test_gpu_special.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
