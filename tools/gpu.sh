#!/bin/bash
# usage: tools/gpu.sh <script-in-repo-root> [timeout_s]  -- runs it on the GPU box
cd /root/repo || exit 1
[ -f "$1" ] || { echo "no such script: $1"; exit 1; }
timeout $(( ${2:-1500} + 1200 )) /usr/local/graft/bin/gpurun --timeout ${2:-1500} -- "bash $1" 2>&1 | tail -3
