# Round-2 evidence, part 2: one ncu --set full capture of C2's, C3's and C5's kernels (C4's is part of
# tools/gpu_round2_evidence.sh); raw pages exported next to the reports.
O=gpurun_out/prof2
rm -rf $O && mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_contig_tma -s 2 -c 2 -o $O/c2_full python tools/prof_run.py c2 2 > $O/ncu_c2.log 2>&1; echo "c2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_splitk -c 3 -o $O/c3_full python tools/prof_run.py c3 1 > $O/ncu_c3.log 2>&1; echo "c3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cols_tma|k_contig_tma" -c 3 -o $O/c5_full python tools/prof_run.py c5 1 > $O/ncu_c5.log 2>&1; echo "c5 rc=$?"
for c in c2 c3 c5; do ncu -i $O/${c}_full.ncu-rep --page raw --csv > $O/${c}_full_raw.csv 2>/dev/null; done
ls -la $O
# the reports together exceed the 64 MiB copy-back limit: summarise on the box, bring back summaries + raw pages
for c in c2 c3 c5; do python tools/ncu_summary.py report $O/${c}_full.ncu-rep $O/r2_${c}_full.md > /dev/null 2>&1; echo "summary $c rc=$?"; done
rm -f $O/*.ncu-rep
ls -la $O
