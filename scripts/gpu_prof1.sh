cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/prof_estep.py --n 4000 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:estep_cfust -s 1 -c 1 -o gpurun_out/prof_cfg2 python scripts/prof_estep.py --n 4000 > gpurun_out/ncu_full.log 2>&1
echo "exit $?" >> gpurun_out/ncu_full.log
