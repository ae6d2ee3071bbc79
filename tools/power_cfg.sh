# developer: pipeline configurations at the power cap (sustained loops), dev library
export PTDR_LIB_NAME=libptdr_dev.so
for c in 1 4 1 4; do echo "== cfg $c"; PTDR_PIPE_CFG=$c timeout 120 python tools/power_probe.py 2>&1 | grep dense; done
