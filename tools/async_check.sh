timeout 900 python -m pytest tests/test_gpu_async_upload.py tests/test_gpu_solve_system.py tests/test_gpu_ffi.py -x -q 2>&1 | tail -3
for k in 3 4 2; do timeout 300 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/a.json 2>gpurun_out/a.err || tail -3 gpurun_out/a.err
python -c "
import json; d=json.load(open('gpurun_out/a.json')); print('k=$k', '%.1f GF/s %.3f ms' % (d['value'], d['ms_per_step']), 'e2e %.1f (%.3f ms)' % (d['e2e']['value'], d['e2e']['ms_per_step']))"; done
