# r02 call c: bench line (cfg5 default), ncu metrics of one full-size cfg5 E-step (roofline constants),
# ncu --set full on a 1e6-row slice, the launch list of the bench command; optional golden chunk.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/gold
if [ -f tests/golden/fit_cfg2_full.partial.json ]; then
  cp tests/golden/fit_cfg2_full.partial.json gpurun_out/gold/
  (python scripts/make_fit_goldens.py cfg2_full --dir gpurun_out/gold --budget-s ${GOLD_BUDGET:-1500} --threads 10 > gpurun_out/gold/cfg2.log 2>&1) &
  GP=$!
fi
python -m paper_2005_06848_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python bench.py ${BENCH_ARGS:---steps 5 --warmup 3} > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
M="gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.avg.per_cycle_active,launch__registers_per_thread,sm__warps_active.avg.per_cycle_active"
timeout 900 ncu --metrics $M --clock-control none -k regex:estep_cfust -c 1 --csv python scripts/prof_estep.py --config 5 --n 10000000 --full-slice --reps 1 > gpurun_out/ncu_metrics_cfg5.csv 2> gpurun_out/ncu_metrics_cfg5.err
timeout 600 ncu --metrics $M --clock-control none -k regex:estep_cfust -c 1 --csv python scripts/prof_estep.py --config 2 --n 100000 --reps 1 > gpurun_out/ncu_metrics_cfg2.csv 2> gpurun_out/ncu_metrics_cfg2.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:estep_cfust -c 1 -o gpurun_out/prof_cfg5_slice -f python scripts/prof_estep.py --config 5 --n 1000000 --full-slice --reps 1 > gpurun_out/ncu_full_cfg5.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
if [ -n "$FUZZ" ]; then
  for sd in 777 4242 99; do
    CFUST_FUZZ_N=400 CFUST_FUZZ_SEED=$sd timeout 900 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/fuzz_$sd.log 2>&1
  done
fi
if [ -n "$GP" ]; then wait $GP; echo "gold exit $?" >> gpurun_out/gold/cfg2.log; fi
