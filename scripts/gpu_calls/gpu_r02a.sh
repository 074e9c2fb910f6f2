# r02 first call: cfg2 golden chunk on the host cores (background) + the GPU test suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/gold
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
cp tests/golden/fit_cfg2_full.partial.json gpurun_out/gold/ 2>/dev/null
(python scripts/make_fit_goldens.py cfg2_full --dir gpurun_out/gold --budget-s ${GOLD_BUDGET:-1300} --threads $(( $(nproc) - 2 )) > gpurun_out/gold/cfg2.log 2>&1) &
GP=$!
python -m paper_2005_06848_b200.build > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
wait $GP
echo "gold exit $?" >> gpurun_out/gold/cfg2.log
