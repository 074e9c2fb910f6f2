# r02 call i: source-level ncu of the M-step (cfg1, cfg3), the chi-node kernel (cfg1) and the q=0 E-step (cfg3);
# the reports are read on the box (raw + source pages as CSV) and only the CSVs come back
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2005_06848_b200.build > gpurun_out/build.log 2>&1
timeout 300 python scripts/iter_profile.py 3 4 > gpurun_out/iter3.log 2>&1 || exit 1
timeout 300 python scripts/iter_profile.py 1 4 > gpurun_out/iter1.log 2>&1 || exit 1
R=/tmp/r02i; mkdir -p $R
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mstep_fused -s 2 -c 1 -o $R/mstep_cfg3 -f python scripts/iter_profile.py 3 4 > gpurun_out/ncu_m3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mstep_fused|chi_kernel|estep_cfust" -s 6 -c 3 -o $R/iter_cfg1 -f python scripts/iter_profile.py 1 4 > gpurun_out/ncu_m1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:estep_t_mma -s 2 -c 1 -o $R/estep_cfg3 -f python scripts/iter_profile.py 3 4 > gpurun_out/ncu_e3.log 2>&1
for f in mstep_cfg3 iter_cfg1 estep_cfg3; do
  ncu -i $R/$f.ncu-rep --page raw --csv > gpurun_out/r02i_${f}_raw.csv 2>/dev/null
  ncu -i $R/$f.ncu-rep --page source --csv --print-source sass > gpurun_out/r02i_${f}_sass.csv 2>/dev/null
  ncu -i $R/$f.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02i_${f}_cuda.csv 2>/dev/null
  ncu -i $R/$f.ncu-rep --page details --csv > gpurun_out/r02i_${f}_details.csv 2>/dev/null
done
du -sh gpurun_out/*
