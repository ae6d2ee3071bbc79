# developer: chunk-group interleaving of the ticket order (dev library) at the power cap and back to back
export PTDR_LIB_NAME=libptdr_dev.so
for g in 0 1 2 0 1 2; do
  for L in 2 5; do
    echo "== grp=$g L=$L"; PTDR_GRP=$g PTDR_L=$L timeout 120 python tools/power_probe.py 2>&1 | grep dense
  done
done
