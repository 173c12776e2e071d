# A/B: graph node priorities on (default) vs off
for k in 2 3 4; do
for v in "" 1; do
MPCORE_GRAPH_NO_PRIO=$v timeout 300 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/ab.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print($k, 'noprio=$v', '%.1f GF/s %.2f ms' % (d['value'], d['ms_per_step']), 'step %.3f' % d['roofline']['whole_step_frac'])"
done; done
for k in 2 3; do for J in 992 1504; do
echo "== k=$k J=$J"; MPCORE_TRACE_PANEL=$J timeout 120 python tools/panel_trace.py $k 2048 2>&1 | tail -3
done; done
