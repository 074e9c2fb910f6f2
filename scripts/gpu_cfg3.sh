cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "3-" > gpurun_out/t3.log 2>&1
for v in "" _tmb2 _told; do CFUST_LIB=paper_2005_06848_b200/libcfust$v.so python scripts/bench_configs.py --configs 3 --iters 5 >> gpurun_out/cfg3.log 2>&1; done
