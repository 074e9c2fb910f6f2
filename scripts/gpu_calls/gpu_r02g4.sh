# r02: the 1200-case wide fuzz (3 seeds x 400, every pair) on the final build.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for seed in 777 4242 99; do
  CFUST_FUZZ_N=400 CFUST_FUZZ_SEED=$seed timeout 600 python -m pytest tests/test_gpu_fuzz.py -m gpu -q 2>&1 | tail -1 | sed "s/^/seed $seed: /" >> gpurun_out/r02g4_fuzz_wide.log
done
