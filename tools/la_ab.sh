# wide-update efficiency with / without the concurrent look-ahead panel
for v in "" 1; do
MPCORE_NO_LOOKAHEAD=$v timeout 300 python bench.py --k 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/ab.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ab.json')); r=d['roofline']; print('nola=$v', '%.1f GF/s %.2f ms' % (d['value'], d['ms_per_step']), 'upd frac %.3f step %.3f' % (r['frac'], r['whole_step_frac']), {a: round(b,2) for a,b in d['kernels_ms_per_step'].items()})"
done
