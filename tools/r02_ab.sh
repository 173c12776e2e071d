#!/bin/bash
cd "$GRAFT_REPO_ROOT"
echo "=== round-1 library"
MPCORE_LIB=$PWD/build/alt/libmpcore_r1.so REPS=3 timeout 500 python tools/onecall_check.py 16384 32768
echo "=== current library"
REPS=3 timeout 500 python tools/onecall_check.py 16384 32768
