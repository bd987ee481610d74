# ncu --set full of C4's two kernels (one launch each) with source correlation; the report and the
# raw/source pages come back under gpurun_out/prof_c4
O=gpurun_out/prof_c4
rm -rf $O && mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_splitk|k_cols_tma" -s 2 -c 2 \
  -o $O/c4 python tools/prof_run.py c4 2 > $O/ncu.log 2>&1
echo "ncu rc=$?"
for k in k_splitk k_cols_tma; do
  ncu -i $O/c4.ncu-rep -k regex:$k --page raw --csv > $O/${k}_raw.csv 2>/dev/null
  ncu -i $O/c4.ncu-rep -k regex:$k --page source --csv --print-source sass > $O/${k}_sass.csv 2>/dev/null
  ncu -i $O/c4.ncu-rep -k regex:$k --page details --csv > $O/${k}_details.csv 2>/dev/null
done
ls -la $O
