# r02 call f (= e with small outputs): reports go to /tmp on the box and only summaries / raw CSV come back
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2005_06848_b200.build > gpurun_out/build.log 2>&1
timeout 600 python scripts/iter_time.py --configs 1,3 > gpurun_out/iter_time.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_nccl1.csv python scripts/nccl1_fit.py 1 > gpurun_out/nccl1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mstep_fused|chi_kernel|estep_t_mma" -c 3 -o /tmp/prof_small -f python scripts/prof_estep.py --config 3 --n 4000000 --reps 1 --em-iters 1 > gpurun_out/ncu_small.log 2>&1
ncu -i /tmp/prof_small.ncu-rep --page raw --csv > gpurun_out/prof_small_raw.csv 2>/dev/null
ncu -i /tmp/prof_small.ncu-rep --page details > gpurun_out/prof_small_details.txt 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"estep_cfust|chi_kernel|mstep_fused" -c 4 -o /tmp/prof_cfg1 -f python scripts/prof_estep.py --config 1 --n 1000 --reps 1 --em-iters 1 > gpurun_out/ncu_cfg1.log 2>&1
ncu -i /tmp/prof_cfg1.ncu-rep --page raw --csv > gpurun_out/prof_cfg1_raw.csv 2>/dev/null
ncu -i /tmp/prof_cfg1.ncu-rep --page details > gpurun_out/prof_cfg1_details.txt 2>/dev/null
M="gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.avg.per_cycle_active,launch__registers_per_thread,sm__warps_active.avg.per_cycle_active"
timeout 1500 ncu --replay-mode application --metrics $M --clock-control none -k regex:estep_cfust -c 1 --csv python scripts/prof_estep.py --config 5 --n 10000000 --full-slice --reps 1 > gpurun_out/ncu_metrics_cfg5.csv 2> gpurun_out/ncu_metrics_cfg5.err
timeout 2400 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
du -sh gpurun_out
