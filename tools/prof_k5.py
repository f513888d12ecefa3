"""K5 timing: tcgen05 projection + fused K1 vs torch GEMM (cuBLAS) + K1.

    python tools/prof_k5.py [R] [V] [K] [M]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_02164_b200.search import proj_lse_topm, row_lse_topm  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1300
V = int(sys.argv[2]) if len(sys.argv) > 2 else 42024
K = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
M = int(sys.argv[4]) if len(sys.argv) > 4 else 5
h = (torch.randn(R, K, device="cuda") * 0.5).to(torch.bfloat16)
w = (torch.randn(V, K, device="cuda") / 16).to(torch.bfloat16)
out = torch.empty(R, V, device="cuda", dtype=torch.bfloat16)


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


t5 = timeit(lambda: proj_lse_topm(h, w, M, eos=2))
tg = timeit(lambda: torch.matmul(h, w.T, out=out))
tk1 = timeit(lambda: row_lse_topm(out, M))
fl = 2.0 * R * V * K
print(f"R={R} V={V} K={K}: K5 {t5:.1f} us ({fl / t5 / 1e6:.0f} TFLOP/s) | cuBLAS {tg:.1f} us ({fl / tg / 1e6:.0f} TFLOP/s) + K1 {tk1:.1f} us "
      f"= {tg + tk1:.1f} us")
