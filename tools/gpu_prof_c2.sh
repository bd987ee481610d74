# ncu --set full of C2's two kernels (forward, inverse) and the register-only calibration loop
O=gpurun_out/prof_c2
rm -rf $O && mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_contig_tma" -s 2 -c 2 \
  -o $O/c2 python tools/prof_run.py c2 2 > $O/ncu.log 2>&1
echo "ncu c2 rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"k_calib" -s 1 -c 1 -o $O/calib \
  python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_calib.log 2>&1
echo "ncu calib rc=$?"
for k in k_contig_tma; do
  ncu -i $O/c2.ncu-rep -k regex:$k --page raw --csv > $O/${k}_raw.csv 2>/dev/null
  ncu -i $O/c2.ncu-rep -k regex:$k --page source --csv --print-source sass > $O/${k}_sass.csv 2>/dev/null
done
ncu -i $O/calib.ncu-rep --page raw --csv > $O/calib_raw.csv 2>/dev/null
ncu -i $O/calib.ncu-rep --page source --csv --print-source sass > $O/calib_sass.csv 2>/dev/null
ls -la $O
