for nt in 256 512 1024; do
  echo "NT $nt"; DPC_SSSP_NT=$nt timeout 300 python tools/lab_sssp.py --scales 16 18 20 --reps 7 2>&1 | grep grid | sed 's/ mean.*iters/ iters/'
done
