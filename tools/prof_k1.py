"""Standalone K1 driver for ncu: full-width WMT step (R=6400 x |V|=42024 bf16)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_02164_b200.search import row_lse_topm  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 6400
V = int(sys.argv[2]) if len(sys.argv) > 2 else 42024
M = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dt = torch.float32 if (len(sys.argv) > 4 and sys.argv[4] == "f32") else torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
u = torch.rand((R, V), device="cuda", generator=g).clamp_min_(2.0 ** -24)
x = (-0.5 * torch.log2(u)).to(dt)
del u
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(6):
    flush.fill_(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    row_lse_topm(x, M)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("K1 ms per launch:", [round(t, 4) for t in ts], "GB/s:", round(R * V * x.element_size() / min(ts[2:]) / 1e6, 1))
