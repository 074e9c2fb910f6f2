# usage: bash scripts/gpu_calls/gpu_cfg3.sh name1 name2 ...  (paper_2005_06848_b200/libcfust_<name>.so)
# q = 0 parity for each build, then the cfg3 E-step time (3 repetitions) -> gpurun_out/cfg3.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" >> gpurun_out/cfg3.log
  CFUST_LIB=paper_2005_06848_b200/libcfust_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "3-" 2>&1 | tail -1 >> gpurun_out/cfg3.log
done
for r in 1 2 3; do
  for v in "$@"; do
    CFUST_LIB=paper_2005_06848_b200/libcfust_$v.so python scripts/bench_configs.py --configs 3 --iters 5 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', 'estep_ms', round(d['estep_ms'],4))" >> gpurun_out/cfg3.log
  done
done
