# r02 call g: full GPU suite, default bench, small-config iteration times, bench launch list, NCCL launch sequence
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2005_06848_b200.build > gpurun_out/build.log 2>&1
timeout 600 python scripts/iter_time.py --configs 1,3 > gpurun_out/iter_time.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_nccl1.csv python scripts/nccl1_fit.py 1 > gpurun_out/nccl1.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
timeout 3000 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 > gpurun_out/bench_ncu.log 2>&1
du -sh gpurun_out
