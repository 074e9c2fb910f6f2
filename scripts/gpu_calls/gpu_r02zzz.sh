# r02 final call: the default bench (cfg5) of the final build with the refreshed roofline constants, its launch
# list, and the reference arm (oracle on the box's host cores) for the record.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02f_nvsmi.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02f_bench_cfg5.log 2> gpurun_out/r02f_bench_cfg5.err; echo "bench exit $?" >> gpurun_out/r02f_bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_bench_reference.log 2> gpurun_out/r02f_bench_reference.err; echo "bench exit $?" >> gpurun_out/r02f_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches_bench_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_ncu_bench.log 2>&1; echo "ncu exit $?" >> gpurun_out/r02f_ncu_bench.log
