# per-stage cost of the on-chip kernels at the row-pass sizes (8 GiB batches of u64)
P=4179340454199820289
for spec in "x:$P:64:15:32768:fwd" "x:$P:64:14:65536:fwd" "x:$P:64:13:131072:fwd" "x:$P:64:12:262144:fwd"; do
  timeout 300 python tools/time_cfg.py $spec 10
done
