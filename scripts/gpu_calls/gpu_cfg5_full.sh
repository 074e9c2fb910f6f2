# cfg5 at full size (n = 1e7): Q3 NP 1 (q3n1) vs the default build, interleaved, with SM clock /
# power samples taken during the runs -> gpurun_out/cfg5_full.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader -lms 500 > gpurun_out/cfg5_smi.log 2>&1 &
SMI=$!
for r in 1 2; do
  for v in q3n1 cur; do
    lib=paper_2005_06848_b200/libcfust_$v.so; [ "$v" = cur ] && lib=paper_2005_06848_b200/libcfust.so
    echo "== $v $(date +%s.%N)" >> gpurun_out/cfg5_full.log
    CFUST_LIB=$lib timeout 600 python scripts/prof_estep.py --config 5 --n 10000000 --reps 1 2>&1 >> gpurun_out/cfg5_full.log
  done
done
kill $SMI
