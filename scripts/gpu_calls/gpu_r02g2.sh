# r02 call after the final bench: one-point-ahead loads in sov_direct (SOV-direct estimator, CFUST_PFD_MASK):
# cur = off (shipped), pfd = q 1..6; E-step ms with estimator = direct, 2 rounds; then the direct-estimator parity
# tests against the pfd build (bitwise-equal results are expected: loads only).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do
  for spec in "5 2000000" "2 100000" "4 200000" "1 200000"; do
    set -- $spec
    for v in cur pfd; do
      lib=paper_2005_06848_b200/libcfust_$v.so; [ "$v" = cur ] && lib=paper_2005_06848_b200/libcfust.so
      CFUST_LIB=$lib timeout 300 python scripts/prof_estep.py --estimator direct --config $1 --n $2 --reps 2 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/r02g2_ab_direct.log
    done
  done
done
CFUST_LIB=paper_2005_06848_b200/libcfust_pfd.so timeout 900 python -m pytest tests -m gpu -q -k "direct or fuzz or smoke" > gpurun_out/r02g2_pytest_pfd.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02g2_pytest_pfd.log
