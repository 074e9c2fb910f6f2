# r02 last call: final build (sov_direct one-point-ahead loads on): smoke, the full GPU suite, SOV-direct E-step times.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g3_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02g3_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/r02g3_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02g3_pytest_gpu.log
for spec in "5 2000000" "2 100000"; do set -- $spec
  timeout 300 python scripts/prof_estep.py --estimator direct --config $1 --n $2 --reps 2 2>&1 | tail -1 >> gpurun_out/r02g3_direct.log
  timeout 300 python scripts/prof_estep.py --config $1 --n $2 --reps 2 2>&1 | tail -1 >> gpurun_out/r02g3_direct.log
done
