#!/bin/bash
# Rebuild the in-tree extension, then run a command on the GPU box (the .so travels with the snapshot).
set -e
cd /root/repo
python paper_2505_10168_b200/build.py > /dev/null
exec /usr/local/graft/bin/gpurun "$@"
