#!/bin/bash
# Box survey: CPU, RAM, storage, PCIe link, host-link copy rates.
mkdir -p gpurun_out
{
echo "== nproc"; nproc
echo "== lscpu"; lscpu | head -30
echo "== numa"; ls /sys/devices/system/node/ | grep node; cat /sys/devices/system/node/node*/meminfo 2>/dev/null | grep MemTotal
echo "== free"; free -g
echo "== hugepages"; grep -i huge /proc/meminfo
echo "== ulimit -l"; ulimit -l
echo "== df"; df -h / /tmp /dev/shm . 2>/dev/null
echo "== mounts"; mount | grep -E ' / | /tmp | /root|nvme|shm' | head
echo "== lsblk"; lsblk 2>/dev/null | head -30
echo "== nvidia-smi"; nvidia-smi
echo "== topo"; nvidia-smi topo -m
echo "== pcie"; nvidia-smi -q | grep -A 12 -E "GPU Link Info|PCIe Generation" | head -40
echo "== dd tmp"; dd if=/dev/zero of=/tmp/ddtest bs=64M count=64 conv=fdatasync 2>&1 | tail -1; rm -f /tmp/ddtest
echo "== dd repo"; dd if=/dev/zero of=./ddtest bs=64M count=64 conv=fdatasync 2>&1 | tail -1; rm -f ./ddtest
echo "== dd shm"; dd if=/dev/zero of=/dev/shm/ddtest bs=64M count=32 2>&1 | tail -1; rm -f /dev/shm/ddtest
echo "== probe"; ./tools/probe/probe
} > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt | tail -80
