# LU bench per forced GEMM tile (MPCORE_GEMM_TILE) vs the chooser (-1)
for k in ${KS:-3 2}; do for t in -1 0 1 2 3 5; do
MPCORE_GEMM_TILE=$t timeout 300 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/t.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/t.json')); print($k, $t, '%.1f GF/s %.2f ms' % (d['value'], d['ms_per_step']), {a: round(b,2) for a,b in d['kernels_ms_per_step'].items()})"
done; done
