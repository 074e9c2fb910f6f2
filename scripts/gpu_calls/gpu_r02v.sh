# r02 call v (re-entry check of HEAD): smoke, full GPU suite, default bench (cfg5), bench launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02v_nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02v_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02v_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02v_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02v_bench.log 2> gpurun_out/r02v_bench.err; echo "bench exit $?" >> gpurun_out/r02v_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02v_launches_bench_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02v_ncu_bench.log 2>&1; echo "ncu exit $?" >> gpurun_out/r02v_ncu_bench.log
