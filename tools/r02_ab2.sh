#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for v in current v2 nograph; do
  echo "=== $v"
  case $v in
    current) timeout 400 python tools/seq_ab.py ;;
    v2) MPCORE_LIB=$PWD/build/alt/libmpcore_v2.so timeout 400 python tools/seq_ab.py ;;
    nograph) MPCORE_NO_GRAPH=1 timeout 400 python tools/seq_ab.py ;;
  esac
done 2>&1 | grep -v Warning
