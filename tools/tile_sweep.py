"""Issue efficiency of each GEMM tile candidate at a many-wave update shape
(C += (-A) B with KK = 32, M = N large), per precision.
usage: [TILES="0 1 8"] [KS="2"] tile_sweep.py [M] [KK]   (spawns one process per candidate, since
MPCORE_GEMM_TILE is read once per process)"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MADD = {2: 29, 3: 214, 4: 326}

def child(M, KK):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2107_12550_b200 import _native as nat
    L = nat.lib()
    dadd, _ = nat.fp64_peak()
    out = {}
    for k in [int(v) for v in os.environ.get("KS", "2 3 4").split()]:
        A = torch.rand(k, M, KK, dtype=torch.float64, device="cuda")
        B = torch.rand(k, KK, M, dtype=torch.float64, device="cuda")
        C = torch.rand(k, M, M, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        def run():
            nat.check(L.mpcore_dev_gemm(k, 1, 0, M, M, KK, A.data_ptr(), KK, M * KK,
                                        B.data_ptr(), M, KK * M, C.data_ptr(), M,
                                        M * M), "gemm")
        run()
        nat.prof_enable(True); nat.prof_reset()
        for _ in range(3):
            run()
        ms, cnt = nat.prof_read()["gemm"]
        nat.prof_enable(False)
        t = ms / cnt / 1e3
        out[k] = M * M * KK * MADD[k] / t / dadd
        del A, B, C
        torch.cuda.empty_cache()
    print(json.dumps(out))

if __name__ == "__main__":
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    KK = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    if os.environ.get("TILE_SWEEP_CHILD"):
        child(M, KK); sys.exit(0)
    for i in [int(v) for v in os.environ.get("TILES", "0 1 2 3 4 5").split()]:
        env = dict(os.environ, MPCORE_GEMM_TILE=str(i), TILE_SWEEP_CHILD="1")
        r = subprocess.run([sys.executable, __file__, str(M), str(KK)], env=env,
                           capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
        print("tile %d: %s" % (i, line), flush=True)
