# developer: L2 policies / store hints at the power cap (sustained loops)
echo "== product"; timeout 120 python tools/power_probe.py 2>&1 | grep dense
for P in nnn fln fnl; do echo "== dev PTDR_POL=$P"; PTDR_LIB_NAME=libptdr_dev.so PTDR_POL=$P timeout 120 python tools/power_probe.py 2>&1 | grep dense; done

