# SSSP stream form: L2 bulk prefetch of each window item's slice (DPC_SSST_PF bytes), scales 22 / 24
for r in 1 2; do
for v in 0 8192 65536; do
  echo "== DPC_SSST_PF=$v"
  DPC_SSST_PF=$v python tools/lab_sssp.py --scales 22 24 --reps 5 | grep grid
done
done
