# r02 call zz (final build: one-block-ahead loads at q = 3 and q = 4): cfg2 ncu metrics (roofline constants),
# smoke, the full GPU suite, the cfg2 bench line.  The cfg5 (q = 3) kernel is the one call z measured.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
M="gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.avg.per_cycle_active,launch__registers_per_thread,sm__warps_active.avg.per_cycle_active"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02zz_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02zz_smoke.log
timeout 600 python scripts/prof_estep.py --config 2 --n 100000 --reps 2 > gpurun_out/r02zz_prof_cfg2.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:estep_cfust -c 1 --csv python scripts/prof_estep.py --config 2 --n 100000 --reps 1 > gpurun_out/r02zz_ncu_metrics_cfg2.csv 2> gpurun_out/r02zz_ncu_metrics_cfg2.err
timeout 1500 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/r02zz_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02zz_pytest_gpu.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/r02zz_bench_cfg2.log 2> gpurun_out/r02zz_bench_cfg2.err; echo "bench exit $?" >> gpurun_out/r02zz_bench_cfg2.err
