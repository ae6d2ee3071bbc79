# developer: host<->device copy rates with and without binding to the GPU's local CPUs/NUMA node
nvidia-smi topo -m 2>/dev/null | head -5
BUS=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//; s/^/0000/')
echo "bus=$BUS"
ls /sys/bus/pci/devices/ | grep -i "${BUS#0000}" | head -2
DEV=/sys/bus/pci/devices/$(ls /sys/bus/pci/devices/ | grep -i "${BUS:4}" | head -1)
echo "local_cpulist=$(cat $DEV/local_cpulist 2>/dev/null) numa_node=$(cat $DEV/numa_node 2>/dev/null)"
lscpu | grep -i "numa\|socket" | head -5
echo -n "unbound: "; python tools/e2e_breakdown.py
CPUS=$(cat $DEV/local_cpulist 2>/dev/null)
if [ -n "$CPUS" ]; then echo -n "bound to $CPUS: "; taskset -c $CPUS python tools/e2e_breakdown.py; fi
NODE=$(cat $DEV/numa_node 2>/dev/null)
if [ -n "$NODE" ] && [ "$NODE" -ge 0 ] && command -v numactl >/dev/null; then echo -n "numactl node $NODE: "; numactl --cpunodebind=$NODE --membind=$NODE python tools/e2e_breakdown.py; fi
