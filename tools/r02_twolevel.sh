#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for k in 3 4 2; do timeout 600 python tools/twolevel_ab.py $k 2048 64 128 256; done
timeout 600 python tools/twolevel_ab.py 2 8192 128 256 512
