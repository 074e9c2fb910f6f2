# r02 call q: cfg1 (q = 2, n = 1e3) E-step variants: points per lane per iteration (NP), blocks per SM (MB), forced SPLIT
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in cur np2 mb3 mb4 np2mb3; do
  for sp in 0 2 4 8; do
    CFUST_SPLIT=$sp CFUST_LIB=paper_2005_06848_b200/libcfust_$v.so timeout 120 python scripts/bench_configs.py --configs 1 --iters 20 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v split=$sp estep_ms', round(d['estep_ms'],4), 'mstep_ms', round(d['mstep_ms'],4))" >> gpurun_out/r02q_cfg1.log 2>&1
  done
done
