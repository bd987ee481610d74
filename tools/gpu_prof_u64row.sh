# ncu --set full of the u64 2^15 cluster row pass (C4's row-pass shape) for the library in NTT_B200_LIB
# (default: in-tree); report + raw / SASS pages under gpurun_out/$OUT
O=gpurun_out/${OUT:-prof_u64row}
rm -rf $O && mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_splitk -s 2 -c 1 \
  -o $O/u64 python tools/time_cfg.py x:4179340454199820289:64:15:2048:fwd 1 > $O/u64.log 2>&1; echo "ncu u64 rc=$?"
ncu -i $O/u64.ncu-rep --page raw --csv > $O/u64_raw.csv 2>/dev/null
ncu -i $O/u64.ncu-rep --page source --csv --print-source sass > $O/u64_sass.csv 2>/dev/null
ls -la $O
