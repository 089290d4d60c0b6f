for f in 0 1 2 3; do
  echo "form $f"; DPC_SSST_FORM=$f timeout 300 python tools/lab_sssp.py --scales 22 24 --reps 3 2>&1 | grep "grid" | sed 's/ mean.*iters/ iters/'
done
