# ncu --set full captures (one launch per kernel) of C2, C3 and the u64 row-pass shape with source pages,
# for the per-instruction shared-memory excess-wavefront scan (tools/smem_excess.py)
O=gpurun_out/${OUT:-conf}
rm -rf $O && mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_contig_tma -s 2 -c 2 \
  -o $O/c2 python tools/prof_run.py c2 2 > $O/c2.log 2>&1; echo "c2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_splitk -c 3 \
  -o $O/c3 python tools/prof_run.py c3 1 > $O/c3.log 2>&1; echo "c3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_splitk -s 2 -c 1 \
  -o $O/u64 python tools/time_cfg.py x:4179340454199820289:64:15:2048:fwd 1 > $O/u64.log 2>&1; echo "u64 rc=$?"
for r in c2 c3 u64; do
  ncu -i $O/$r.ncu-rep --page source --csv --print-source sass > $O/${r}_sass.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
ls -la $O
