cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/exp2.log; : > $out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown --format=csv -lms 100 > gpurun_out/exp2_clocks.csv &
SMI=$!
for n in 4000 20000 100000 100000; do python scripts/prof_estep.py --n $n --reps 3 >> $out 2>&1; done
kill $SMI
python scripts/prof_estep.py --n 4000 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:estep_cfust -s 1 -c 1 -o gpurun_out/prof_cfg2_np1 -f python scripts/prof_estep.py --n 4000 > gpurun_out/ncu_full.log 2>&1
