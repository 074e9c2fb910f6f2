cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/bench_configs.py > gpurun_out/configs.log 2>&1
python scripts/prof_estep.py --config 3 --n 400000 > gpurun_out/prof_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:estep_t -s 1 -c 1 -o gpurun_out/prof_cfg3 -f python scripts/prof_estep.py --config 3 --n 400000 > gpurun_out/ncu3.log 2>&1
