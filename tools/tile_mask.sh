# LU bench per update-tile candidate mask (MPCORE_UPDATE_TILES)
for k in ${KS:-3 4 2}; do for m in ${MASKS:-0x3f 0x1e 0x0e 0x0c 0x08 0x2e 0x3e}; do
MPCORE_UPDATE_TILES=$m timeout 300 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/t.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/t.json')); print($k, '$m', '%.1f GF/s %.2f ms' % (d['value'], d['ms_per_step']), {a: round(b,2) for a,b in d['kernels_ms_per_step'].items()})"
done; done
