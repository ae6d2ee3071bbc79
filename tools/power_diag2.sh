for L in libptdr.so libptdr_diag1.so libptdr_diag2.so; do
  echo "== $L"; PTDR_LIB_NAME=$L timeout 120 python tools/power_probe.py 2>&1 | grep dense
done
