#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 300 python tools/conv_dbg.py 2>&1 | tail -20
MPCORE_REFINE_TIMERS=1 timeout 300 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu 2>&1 >/dev/null | grep -i "convert\|flat" 
