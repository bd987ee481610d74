# ncu --set full of the split kernels (C3's three u32 launches of one prime, C4's u64 row pass) with
# source correlation; per-CUDA-line and per-SASS-line stall pages come back under gpurun_out/$OUT
O=gpurun_out/${OUT:-prof_src}
rm -rf $O && mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_splitk -c 3 \
  -o $O/c3 python tools/prof_run.py c3 1 > $O/c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_splitk -s 2 -c 1 \
  -o $O/u64 python tools/time_cfg.py x:4179340454199820289:64:15:2048:fwd 1 > $O/u64.log 2>&1; echo "ncu u64 rc=$?"
for r in c3 u64; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page source --csv --print-source sass > $O/${r}_sass.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page source --csv --print-source cuda > $O/${r}_cuda.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null
done
ls -la $O
