set -x
mkdir -p gpurun_out/final
for k in 3 4 2; do timeout 600 python bench.py --k $k --steps 5 --warmup 3 --no-cpu > gpurun_out/final/c2_k$k.json 2> gpurun_out/final/c2_k$k.err; done
for k in 2 3 4; do timeout 600 python bench.py --config 1 --k $k --steps 3 --warmup 2 --no-cpu > gpurun_out/final/c1_k$k.json 2> gpurun_out/final/c1_k$k.err; done
timeout 600 python bench.py --config 3 --steps 5 --warmup 2 > gpurun_out/final/c3.json 2> gpurun_out/final/c3.err
timeout 900 python bench.py --config 4 --dim 8192 --steps 2 --warmup 1 > gpurun_out/final/c4_8192.json 2> gpurun_out/final/c4_8192.err
timeout 1200 python bench.py --config 4 --steps 2 --warmup 1 > gpurun_out/final/c4_32768.json 2> gpurun_out/final/c4_32768.err
timeout 900 python bench.py > gpurun_out/final/default.json 2> gpurun_out/final/default.err
bash tools/profile_round.sh > gpurun_out/final/prof.log 2>&1
ls gpurun_out/prof
