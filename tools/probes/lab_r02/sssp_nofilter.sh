# SSSP level form: distance-filter skip threshold sweep (config 1 + scale 20), interleaved
for r in 1 2; do
for v in 0 16384 65536 262144 1048576; do
  echo "== DPC_SSSP_NOFILTER=$v"
  DPC_SSSP_NOFILTER=$v python tools/lab_sssp.py --scales 16 20 --reps 20 | grep grid
done
done
