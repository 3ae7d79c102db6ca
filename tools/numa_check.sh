#!/bin/bash
# host topology + e2e under CPU binding to each NUMA node
cd /root/repo
mkdir -p gpurun_out
{
lscpu | grep -Ei "model name|socket|numa|^cpu\(s\)"
nvidia-smi topo -m
bdf=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//')
echo "gpu bdf $bdf"
ls /sys/bus/pci/devices/ | grep -i "${bdf#0000}" | while read d; do echo "numa_node $(cat /sys/bus/pci/devices/$d/numa_node) local_cpulist $(cat /sys/bus/pci/devices/$d/local_cpulist)"; done
which taskset numactl
} > gpurun_out/topo.txt 2>&1
for n in $(ls -d /sys/devices/system/node/node* | sed 's/.*node//'); do
  cpus=$(cat /sys/devices/system/node/node$n/cpulist)
  echo "node $n cpus $cpus" >> gpurun_out/numa_e2e.txt
  taskset -c $cpus timeout 300 python tools/e2e_probe.py c5 >> gpurun_out/numa_e2e.txt 2>&1
  taskset -c $cpus timeout 120 python tools/pcie_probe.py 2 >> gpurun_out/numa_e2e.txt 2>&1
done
