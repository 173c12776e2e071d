# per-phase panel traces in situ (DD and TD, n=2048) at several panels
for k in 2 3; do for J in 0 992 1504 1920; do
echo "== k=$k J=$J"; MPCORE_TRACE_PANEL=$J timeout 120 python tools/panel_trace.py $k 2048 2>&1 | tail -9
done; done
