for sc in 22 24; do
  for p in 0 1; do
    DPC_SSSP_PERSIST=$p timeout 300 python tools/lab_sssp.py --scales $sc --reps 3 2>&1 | grep -E "grid|persist"
  done
done
