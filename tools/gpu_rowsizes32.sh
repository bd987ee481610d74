# per-butterfly cost of the u32 kernels by size (1 GiB batches): on-chip 2^12..2^15, 2-CTA cluster 2^16
P=998244353
for spec in "x:$P:32:16:4096:fwd,inv" "x:$P:32:15:8192:fwd,inv" "x:$P:32:14:16384:fwd,inv" "x:$P:32:13:32768:fwd,inv" "x:$P:32:12:65536:fwd,inv"; do
  timeout 300 python tools/time_cfg.py $spec 10
done
