#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 600 python tools/dist_check.py 2048 8192 16384 23000 32768
echo "--- serial"
MPCORE_DIST_SERIAL=1 timeout 600 python tools/dist_check.py 16384 32768
echo "--- no graph"
MPCORE_NO_GRAPH=1 timeout 600 python tools/dist_check.py 32768
