"""Standalone K1 timing / ncu driver: R rows x |V| logits (log-like values).

    python tools/prof_k1.py [R] [V] [M] [f32|bf16] [--noflush] [--legacy] [--b2b]

Outputs are pre-allocated and K1 is launched through the C-ABI directly, so
the CUDA events bracket only the kernel (an L2-flush kernel runs before each
timed launch unless --noflush).
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_02164_b200 import _native as N  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
R = int(args[0]) if len(args) > 0 else 6400
V = int(args[1]) if len(args) > 1 else 42024
M = int(args[2]) if len(args) > 2 else 5
f32 = len(args) > 3 and args[3] == "f32"
flush_between = "--noflush" not in sys.argv
dt = torch.float32 if f32 else torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
u = torch.rand((R, V), device="cuda", generator=g).clamp_min_(2.0 ** -24)
x = (-0.5 * torch.log2(u)).to(dt)
del u
tok = torch.empty((R, M), dtype=torch.int32, device="cuda")
lp = torch.empty((R, M), dtype=torch.float32, device="cuda")
lse = torch.empty((R,), dtype=torch.float32, device="cuda")
fb = torch.zeros((1,), dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
lib = N.load_library()
code = N.VS_DTYPE_F32 if f32 else N.VS_DTYPE_BF16
stream = torch.cuda.current_stream().cuda_stream


legacy = "--legacy" in sys.argv
nbytes = int(lib.vs_row_lse_topm_ws_bytes(R, V, code))
ws = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device="cuda")


def launch():
    if legacy:
        N.check(lib.vs_row_lse_topm(x.data_ptr(), code, x.stride(0), V, M, R, None, R, tok.data_ptr(),
                                    lp.data_ptr(), lse.data_ptr(), fb.data_ptr(), stream), "k1")
    else:
        pin = N.VS_K1_SPLIT if "--split" in sys.argv else 0
        N.check(lib.vs_row_lse_topm_ws(x.data_ptr(), code | pin, x.stride(0), V, M, R, None, R, tok.data_ptr(),
                                       lp.data_ptr(), lse.data_ptr(), fb.data_ptr(), ws.data_ptr(),
                                       ws.numel(), stream), "k1")


if "--b2b" in sys.argv:  # back-to-back launches (inputs > L2), no flush, no host gaps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(12)]
    launch()
    for e0, e1 in evs:
        e0.record()
        launch()
        e1.record()
    torch.cuda.synchronize()
    ts = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
    med = ts[len(ts) // 2]
    print("K1 b2b ms per launch (sorted):", [round(t, 4) for t in ts], "GB/s:",
          round(R * V * x.element_size() / med / 1e6, 1), "fallbacks:", int(fb.item()))
    sys.exit(0)
ts = []
for i in range(8):
    if flush_between:
        flush.fill_(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launch()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
best = min(ts[2:])
print("K1 ms per launch:", [round(t, 4) for t in ts], "GB/s:",
      round(R * V * x.element_size() / best / 1e6, 1), "fallbacks:", int(fb.item()))
