# column count from which TD/QD exchange+U12 uses two columns per warp
for k in ${KS:-3 4}; do for c in ${CS:-0 600 1200 100000}; do
MPCORE_TRSM_PAIR_COLS=$c timeout 300 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/t.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/t.json')); print($k, 'pair>=$c', '%.1f GF/s %.2f ms' % (d['value'], d['ms_per_step']), {a: round(b,2) for a,b in d['kernels_ms_per_step'].items()})"
done; done
