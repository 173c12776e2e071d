mkdir -p gpurun_out/prof
python tools/gemm_bench.py 2048 3 2>&1 | tail -3
for t in 0 1; do
MPCORE_GEMM_TILE=$t timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 1 -c 1 -o gpurun_out/prof/ddgemm_t$t python -c "
import sys; sys.path.insert(0,'.')
from paper_2107_12550_b200 import _native as nat
from paper_2107_12550_b200.linalg import DeviceMatrix
L=nat.lib(); k=2; n=2048
A=DeviceMatrix(k,n,n); A.generate(0,n,1); B=DeviceMatrix(k,n,n); B.generate(1,n,1); C=DeviceMatrix(k,n,n)
for _ in range(3): nat.check(L.mpcore_mat_mul(A.handle,B.handle,C.handle),'mm')
" > gpurun_out/prof/ddgemm_t$t.log 2>&1
done
ls -la gpurun_out/prof
