timeout 900 python -m pytest tests/test_gpu_async_upload.py tests/test_gpu_ffi.py tests/test_gpu_api.py -x -q 2>&1 | tail -2
for k in 2 3 4; do timeout 600 python bench.py --config 1 --k $k --steps 3 --warmup 2 --no-cpu > gpurun_out/a1.json 2>gpurun_out/a1.err || tail -3 gpurun_out/a1.err
python -c "
import json; d=json.load(open('gpurun_out/a1.json')); print('gemm k=$k', '%.1f GF/s %.3f ms' % (d['value'], d['ms_per_step']), 'e2e %.1f' % d['e2e']['value'])"; done
