#!/usr/bin/env bash
# Host facts of a gpurun box (cores, RAM, cgroup limit, CPU model, GPU) -> stdout.
nproc; free -g; cat /sys/fs/cgroup/memory.max 2>/dev/null; grep -m1 "model name" /proc/cpuinfo
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
