for p in 0 8 32 100; do
MPCORE_POLL_NS=$p MPCORE_TRACE_PANEL=0 python tools/panel_trace.py 2 2048 | grep -E "period \(cycles|kernel stamps" | sed "s/^/poll_ns=$p /"
MPCORE_POLL_NS=$p timeout 300 python bench.py --k 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/t.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/t.json')); print('poll_ns=$p', '%.1f GF/s %.2f ms' % (d['value'], d['ms_per_step']))"
done
