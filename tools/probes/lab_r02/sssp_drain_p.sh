# SSSP level form: items per drain step (P = 1 / 2; p2b = P 2 held to 3 blocks / SM), config 1 + scale 20
for r in 1 2; do
for L in old p1 p2 p2b; do
  echo "== $L"
  DPC_LIB_PATH=tools/probes/ab/libdpc_$L.so python tools/lab_sssp.py --scales 16 20 --reps 20 | grep grid
done
done
