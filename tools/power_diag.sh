# developer: power/clock/time of the dense kernel's diagnostic builds at the power cap
for L in libptdr.so libptdr_diag4.so libptdr_diag48.so libptdr_diag52.so; do
  echo "== $L"; PTDR_LIB_NAME=$L timeout 120 python tools/power_probe.py 2>&1 | grep dense
done
