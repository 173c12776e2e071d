for k in ${KS:-2 3}; do for so in 0 64 128 192 256; do
MPCORE_PANEL_SOLO=$so timeout 300 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/t.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/t.json')); print($k, 'solo<=$so', '%.1f GF/s %.2f ms' % (d['value'], d['ms_per_step']), {a: round(b,2) for a,b in d['kernels_ms_per_step'].items()})"
done; done
