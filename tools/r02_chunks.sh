#!/bin/bash
cd "$GRAFT_REPO_ROOT"
MPCORE_REFINE_TIMERS=1 timeout 300 python bench.py --config 3 --steps 1 --warmup 2 --no-cpu 2>&1 >/dev/null | tail -18
