# ncu launch list of the bench command + one full-size --set full capture of the E-step kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
echo "launchlist exit $?" >> gpurun_out/ncu_launch.log
python scripts/prof_estep.py --n 100000 --reps 1 > gpurun_out/prof_full_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:estep_cfust -c 1 -o gpurun_out/prof_cfg2_full -f python scripts/prof_estep.py --n 100000 --reps 1 > gpurun_out/ncu_full2.log 2>&1
echo "full exit $?" >> gpurun_out/ncu_full2.log
