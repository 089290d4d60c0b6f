# H2D / D2H bandwidth of pinned host buffers vs the CPU (NUMA node) that allocates them
lscpu | grep -E "NUMA|Socket|^CPU\(s\)"
bus=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^0000//')
f=$(ls -d /sys/bus/pci/devices/*${bus#0000} 2>/dev/null | head -1)
echo "gpu $bus sysfs $f local_cpulist $(cat $f/local_cpulist 2>/dev/null) numa_node $(cat $f/numa_node 2>/dev/null)"
local=$(cat $f/local_cpulist 2>/dev/null | cut -d, -f1)
echo "== unpinned"; timeout 120 python tools/probes/e2e_batch.py 2>&1 | tail -4
if [ -n "$local" ]; then echo "== taskset -c $local"; timeout 120 taskset -c $local python tools/probes/e2e_batch.py 2>&1 | tail -4; fi
other=$(lscpu | awk -F: '/NUMA node1 CPU/{gsub(/ /,"",$2); print $2}' | cut -d, -f1)
if [ -n "$other" ]; then echo "== taskset -c $other (node 1)"; timeout 120 taskset -c $other python tools/probes/e2e_batch.py 2>&1 | tail -4; fi
