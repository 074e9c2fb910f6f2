# r02 call x: the shipped build (cur = lane-parallel T_1, polynomial exp) against pf1 (one-block-ahead
# chi / W loads with one warp per observation, CFUST_PF1=1) and xt3 (table exp at q = 3, CFUST_SOV_XT=3):
# E-step ms, 2 rounds; then ncu --set full of cur on the cfg5 slice (roofline constants), cfg1 / cfg3
# iteration times, the full GPU suite and the default bench.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do
  for spec in "5 2000000" "1 200000"; do
    set -- $spec
    for v in cur pf1 xt3; do
      lib=paper_2005_06848_b200/libcfust_$v.so; [ "$v" = cur ] && lib=paper_2005_06848_b200/libcfust.so
      CFUST_LIB=$lib timeout 300 python scripts/prof_estep.py --config $1 --n $2 --reps 2 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/r02x_ab.log
    done
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:estep_cfust -s 1 -c 1 -o gpurun_out/r02x_cfg5_slice -f python scripts/prof_estep.py --config 5 --n 1000000 --full-slice --reps 2 > gpurun_out/r02x_ncu.log 2>&1; echo "ncu exit $?" >> gpurun_out/r02x_ncu.log
ncu -i gpurun_out/r02x_cfg5_slice.ncu-rep --page raw --csv > gpurun_out/r02x_ncu_estep_cfg5_slice1e6_raw.csv 2>&1
rm -f gpurun_out/r02x_cfg5_slice.ncu-rep
timeout 600 python scripts/iter_time.py > gpurun_out/r02x_iter_time.log 2>&1; echo "exit $?" >> gpurun_out/r02x_iter_time.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02x_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02x_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02x_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02x_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02x_bench.log 2> gpurun_out/r02x_bench.err; echo "bench exit $?" >> gpurun_out/r02x_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02x_launches_bench_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02x_ncu_bench.log 2>&1; echo "ncu exit $?" >> gpurun_out/r02x_ncu_bench.log
