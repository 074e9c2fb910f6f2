# usage: bash scripts/gpu_calls/gpu_round.sh [tests|bench|prof|all] ; outputs under gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
what=${1:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1; nproc >> gpurun_out/nvsmi.txt
if [[ $what == all || $what == tests ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
  timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
if [[ $what == all || $what == bench ]]; then
  timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
fi
if [[ $what == all || $what == prof ]]; then
  python scripts/prof_estep.py --n 4000 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:estep_cfust -s 1 -c 1 -o gpurun_out/prof_cfg2 -f python scripts/prof_estep.py --n 4000 > gpurun_out/ncu_full.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_full.log
fi
