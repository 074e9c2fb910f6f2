# NVTX ranges of the C ABI seen by ncu: kernels launched inside "cfust:mstep" and "cfust:estep-kernel"
# ranges of a short cfg1 fit (examples/cfust_fit.c path: no Python in the timed process).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
gcc -O2 examples/cfust_fit.c -Iinclude -Lpaper_2005_06848_b200 -lcfust -Wl,-rpath,$PWD/paper_2005_06848_b200 -o /tmp/cfust_fit
python examples/write_problem.py --config 1 /tmp/p1.bin > /dev/null
for r in "cfust:mstep/" "cfust:estep-kernel/" "cfust_fit/"; do
  echo "== nvtx-include $r" >> gpurun_out/nvtx.log
  ncu --nvtx --nvtx-include "$r" --metrics gpu__time_duration.sum --csv /tmp/cfust_fit /tmp/p1.bin 2 2>/dev/null \
    | python -c "
import sys, csv, collections
rows = [r for r in csv.reader(sys.stdin) if len(r) > 5]
h = rows[0]; kn = h.index('Kernel Name'); nv = [i for i, x in enumerate(h) if x.startswith('thread_domain') or 'NVTX' in x or x.startswith('nvtx')]
c = collections.Counter(r[kn].split('(')[0] + '  in ' + ' > '.join(r[i].split(':')[1] for i in nv if ':' in r[i]) for r in rows[1:] if r[0].isdigit())
[print(f'  {v:3d}  {k}') for k, v in sorted(c.items())]" >> gpurun_out/nvtx.log
done
