# r02 call w: A/B of the SOV loop table exp (Tune<Q>::XT, q <= 3) and lane-parallel T_1 (CFUST_T1_LANES):
# cur = both, noxt = T1 lanes only, xtonly = table exp only, base = neither (HEAD e92d5b5 kernel).
# E-step ms on cfg5 / cfg1 slices (2 interleaved rounds), then the q <= 3 parity + special tests with XT
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do
  for spec in "5 2000000" "1 200000" "2 20000"; do
    set -- $spec
    for v in cur noxt xtonly base; do
      lib=paper_2005_06848_b200/libcfust_$v.so; [ "$v" = cur ] && lib=paper_2005_06848_b200/libcfust.so
      CFUST_LIB=$lib timeout 300 python scripts/prof_estep.py --config $1 --n $2 --reps 2 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/r02w_ab.log
    done
  done
done
timeout 1200 python -m pytest tests/test_gpu_special.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_split.py -m gpu -q -x > gpurun_out/r02w_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02w_pytest.log
# ncu --set full of the shipped build's cfg5 E-step on the first 1e6 rows (flops/pair, DRAM bytes, pipes)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:estep_cfust -s 1 -c 1 -o gpurun_out/r02w_cfg5_slice -f python scripts/prof_estep.py --config 5 --n 1000000 --full-slice --reps 2 > gpurun_out/r02w_ncu.log 2>&1; echo "ncu exit $?" >> gpurun_out/r02w_ncu.log
ncu -i gpurun_out/r02w_cfg5_slice.ncu-rep --page raw --csv > gpurun_out/r02w_ncu_estep_cfg5_slice1e6_raw.csv 2>&1
