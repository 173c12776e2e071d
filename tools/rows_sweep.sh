# panel rows-per-CTA target sweep (MPCORE_PANEL_ROWS)
for k in ${KS:-2 3}; do for r in ${ROWS:-24 32 40 48}; do
MPCORE_PANEL_ROWS=$r timeout 300 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/r.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r.json')); print($k, $r, '%.1f GF/s %.2f ms' % (d['value'], d['ms_per_step']), {a: round(b,2) for a,b in d['kernels_ms_per_step'].items()})"
done; done
