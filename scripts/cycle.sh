#!/bin/bash
# build (fail fast) then run a command on the GPU box
set -e
cd /root/repo
python paper_2005_08713_b200/build.py > /tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head; exit 1; }
timeout 2400 /usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-900} -- "$1" 2>&1 | grep -v "^\[gpurun\] \(sending\|merged\)"
