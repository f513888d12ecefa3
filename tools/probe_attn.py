import torch, time
print(torch.cuda.get_device_name())
try:
    import flash_attn
    from flash_attn import flash_attn_with_kvcache
    print("flash_attn", flash_attn.__version__)
    B, Lc, H, D = 6401, 256, 16, 64
    kc = torch.randn(B, Lc, H, D, device="cuda", dtype=torch.bfloat16)
    vc = torch.randn_like(kc)
    R = 573
    q = torch.randn(R, 1, H, D, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(R, 1, H, D, device="cuda", dtype=torch.bfloat16)
    v = torch.randn_like(k)
    idx = torch.randperm(6400, device="cuda")[:R].int()
    sl = torch.randint(1, 60, (R,), device="cuda", dtype=torch.int32)
    o = flash_attn_with_kvcache(q, kc, vc, k=k, v=v, cache_seqlens=sl, cache_batch_idx=idx)
    torch.cuda.synchronize()
    # reference check on row 0
    b = idx[0].item(); L = sl[0].item()
    K = kc[b, :L + 1].float(); V = vc[b, :L + 1].float()
    s = torch.einsum("hd,lhd->hl", q[0, 0].float(), K) / 8.0
    ref = torch.einsum("hl,lhd->hd", s.softmax(-1), V)
    print("fa err", (ref - o[0, 0].float()).abs().max().item(), "k written", torch.equal(kc[b, L], k[0, 0]))
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(20):
        flash_attn_with_kvcache(q, kc, vc, k=k, v=v, cache_seqlens=sl, cache_batch_idx=idx)
    t1.record(); torch.cuda.synchronize(); print("fa us", t0.elapsed_time(t1) / 20 * 1e3)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        flash_attn_with_kvcache(q, kc, vc, k=k, v=v, cache_seqlens=sl, cache_batch_idx=idx)
    g.replay(); torch.cuda.synchronize(); print("graph ok")
except Exception as e:
    import traceback; traceback.print_exc()
try:
    import flashinfer
    print("flashinfer", flashinfer.__version__)
except Exception as e:
    print("flashinfer err", e)
# GEMM timing for decoder step
R, d = 576, 1024
x = torch.randn(R, d, device="cuda", dtype=torch.bfloat16)
W = torch.randn(42024, d, device="cuda", dtype=torch.bfloat16)
for n_ in [3072, 1024, 4096]:
    Wn = torch.randn(n_, d, device="cuda", dtype=torch.bfloat16)
    for _ in range(3): y = x @ Wn.T
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(50): y = x @ Wn.T
    torch.cuda.synchronize(); print("gemm", R, d, n_, (time.perf_counter() - t) / 50 * 1e6, "us")
for _ in range(3): y = x @ W.T
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(20): y = x @ W.T
torch.cuda.synchronize(); print("vocab gemm", (time.perf_counter() - t) / 20 * 1e6, "us")
