#!/bin/bash
# DD/TD panel chain probe: per-panel stamps of one LU and per-phase panel traces
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/s3
out=gpurun_out/s3/panelprobe${TAG}.txt; : > $out
for k in ${KS:-2 3}; do
  echo "== stamps k=$k" >> $out; timeout 120 python tools/lu_stamps.py $k 2048 >> $out 2>&1
  for J in 0 1024 1792; do
    echo "== trace k=$k J=$J" >> $out; MPCORE_TRACE_PANEL=$J timeout 120 python tools/panel_trace.py $k 2048 >> $out 2>&1
  done
done
cat $out
