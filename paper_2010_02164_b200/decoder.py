"""Batched incremental encoder-decoder scorer with a physical-row KV cache.

This is the realistic scorer of SURVEY.md §8(f) row 1 and the consumer of K4
(§8(a) a13).  The reference scorer is stateless: it recomputes from the whole
token tuple (bb/model.py:209-218, bb/core.py:170).  Here each engine physical
row (include/varstream.h) owns a self-attention K/V cache `[layers, 2, n*k,
max_len, d]`:

* a scored row writes K/V at its last position only;
* after the beam step, K2's copy plan (extra children of a parent) is applied
  with `vs_rows_copy` (K4).  First children inherit the parent's row
  untouched;
* admitted sources are encoded and their cross-attention K/V are placed into
  the freed slots with `vs_scatter_rows` (K4's encoder-state half).

Layers run through PyTorch (random init, seeded).  Logits follow SURVEY.md §7
hard part 7: `tau * (h @ W_out^T)` plus an EOS bias `eos_bias * len / src_len`
(like bb/model.py:215), so widths and lengths vary.  The decoder needs R_t on
the host (dynamic GEMM shapes), so it runs under the synchronous driver.
"""

from __future__ import annotations

import ctypes as C
import math

import torch
import torch.nn.functional as F

from . import _native as N
from .core import Vocabulary


class TransformerScorer:
    host_sync = True

    def __init__(self, vocab: Vocabulary, *, d: int = 64, heads: int = 4, layers: int = 2,
                 enc_layers: int = 1, ffn: int = 256, max_src: int = 64, seed: int = 0,
                 tau: float = 4.0, eos_bias: float = 4.0, dtype=torch.float32, device=None,
                 record_logits: bool = False):
        assert d % heads == 0
        self.vocab = vocab
        self.d, self.h, self.nl, self.nel, self.ffn = d, heads, layers, enc_layers, ffn
        self.max_src, self.tau, self.eos_bias, self.dtype = max_src, tau, eos_bias, dtype
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        g = torch.Generator(device="cpu").manual_seed(seed)

        def w(*shape, std=None):
            std = std if std is not None else 1.0 / math.sqrt(shape[-1])
            return (torch.randn(*shape, generator=g) * std).to(self.device, dtype)

        V = vocab.size
        self.emb = w(V, d, std=1.0)
        self.pos = w(512, d, std=0.5)
        self.enc = [dict(qkv=w(3 * d, d), o=w(d, d), f1=w(ffn, d), f2=w(d, ffn)) for _ in range(enc_layers)]
        self.dec = [dict(qkv=w(3 * d, d), o=w(d, d), cq=w(d, d), ckv=w(2 * d, d), co=w(d, d),
                         f1=w(ffn, d), f2=w(d, ffn)) for _ in range(layers)]
        self.out = w(V, d)
        self.record_logits = record_logits
        self.copies = 0  # K4 copies applied (counted when record_logits, sync driver)

    # ------------------------------------------------------------------ model
    def _attn(self, q, k, v, mask):
        # q [B, h, Tq, dh], k/v [B, h, Tk, dh], mask [B, 1, Tq, Tk] bool (True = keep)
        s = (q @ k.transpose(-1, -2)) / math.sqrt(self.d // self.h)
        s = s.masked_fill(~mask, float("-inf"))
        return torch.softmax(s.float(), dim=-1).to(q.dtype) @ v

    def _split(self, x):  # [B, T, d] -> [B, h, T, dh]
        B, T, _ = x.shape
        return x.view(B, T, self.h, self.d // self.h).transpose(1, 2)

    def _merge(self, x):
        B, h, T, dh = x.shape
        return x.transpose(1, 2).reshape(B, T, h * dh)

    def encode_sources(self, src: torch.Tensor, lens: torch.Tensor):
        """src [B, S] int64 (padded), lens [B] -> per decoder layer cross K,V [B, S, d] each."""
        B, S = src.shape
        x = self.emb[src] + self.pos[:S][None]
        keep = (torch.arange(S, device=src.device)[None, :] < lens[:, None])[:, None, None, :]
        for L in self.enc:
            q, k, v = (x @ L["qkv"].T).split(self.d, dim=-1)
            a = self._merge(self._attn(self._split(q), self._split(k), self._split(v), keep))
            x = F.layer_norm(x + a @ L["o"].T, (self.d,))
            x = F.layer_norm(x + F.gelu(x @ L["f1"].T) @ L["f2"].T, (self.d,))
        return [(x @ L["ckv"].T).split(self.d, dim=-1) for L in self.dec]

    def full_forward(self, src_tokens, prefix):
        """Reference (cache-free) logits of the last position of `prefix` given
        `src_tokens` — used by tests to validate the K/V cache + K4 reorder."""
        dev = self.device
        src = torch.tensor([list(src_tokens)], device=dev)
        cross = self.encode_sources(src, torch.tensor([len(src_tokens)], device=dev))
        T = len(prefix)
        x = self.emb[torch.tensor([list(prefix)], device=dev)] + self.pos[:T][None]
        causal = torch.ones(T, T, dtype=torch.bool, device=dev).tril()[None, None]
        ckeep = torch.ones(1, 1, 1, len(src_tokens), dtype=torch.bool, device=dev)
        for L, (ck, cv) in zip(self.dec, cross):
            q, k, v = (x @ L["qkv"].T).split(self.d, dim=-1)
            a = self._merge(self._attn(self._split(q), self._split(k), self._split(v), causal))
            x = F.layer_norm(x + a @ L["o"].T, (self.d,))
            cq = x @ L["cq"].T
            a = self._merge(self._attn(self._split(cq), self._split(ck), self._split(cv), ckeep))
            x = F.layer_norm(x + a @ L["co"].T, (self.d,))
            x = F.layer_norm(x + F.gelu(x @ L["f1"].T) @ L["f2"].T, (self.d,))
        lg = self._project(x[0, -1:])[0].float()
        lg[self.vocab.eos] += self.eos_bias * T / len(src_tokens)
        return lg

    def _project(self, h):
        """Vocab projection (logits before the EOS bias): tau * h @ W_out^T."""
        return (h @ self.out.T).float() * self.tau

    # --------------------------------------------------------- engine protocol
    def bind(self, engine) -> None:
        n, k, Lmax = engine.n, engine.k, engine.max_len
        if Lmax > self.pos.shape[0]:
            raise ValueError("max_len exceeds the decoder's positions")
        dev, dt = engine.device, self.dtype
        self.engine = engine
        # self-attention cache by PHYSICAL row: [layers*2, n*k, max_len, d]
        self.kv = torch.zeros(self.nl * 2, n * k, Lmax, self.d, device=dev, dtype=dt)
        # cross-attention K/V by slot: [n, layers*2, max_src, d]
        self.enc_kv = torch.zeros(n, self.nl * 2, self.max_src, self.d, device=dev, dtype=dt)
        self.enc_len = torch.zeros(n, dtype=torch.long, device=dev)
        self._buf = torch.empty(engine.capacity, self.vocab.size, device=dev, dtype=torch.float32)
        self._corpus_off = engine.t["src_off"].cpu().numpy()
        self._corpus_tok = engine.t["src_tok"].cpu().numpy()

    def on_admit(self, engine, status) -> None:
        n = engine.n
        a0, na = int(status[N.ST_ADMIT0]), int(status[N.ST_NADMIT])
        slots = torch.tensor(status[N.ST_HDR + 3 * n:N.ST_HDR + 3 * n + na].astype("int32"),
                             device=engine.device)
        srcs = [self._corpus_tok[self._corpus_off[i]:self._corpus_off[i + 1]] for i in range(a0, a0 + na)]
        lens = torch.tensor([len(s) for s in srcs], device=engine.device)
        if int(lens.max()) > self.max_src:
            raise ValueError("source longer than the encoder's max_src")
        S = int(lens.max())
        pad = torch.zeros(na, S, dtype=torch.long)
        for i, s in enumerate(srcs):
            pad[i, : len(s)] = torch.from_numpy(s.astype("int64"))
        cross = self.encode_sources(pad.to(engine.device), lens)
        dense = torch.zeros(na, self.nl * 2, self.max_src, self.d, device=engine.device, dtype=self.dtype)
        for li, (ck, cv) in enumerate(cross):
            dense[:, 2 * li, :S] = ck
            dense[:, 2 * li + 1, :S] = cv
        # K4, encoder half: place each admitted source's states into its slot
        N.check(engine.lib.vs_scatter_rows(self.enc_kv.data_ptr(), self.enc_kv.stride(0) * self.enc_kv.element_size(),
                                           dense.data_ptr(), dense.stride(0) * dense.element_size(),
                                           dense.stride(0) * dense.element_size(), slots.data_ptr(), None,
                                           na, engine.stream_ptr), "vs_scatter_rows")
        self.enc_len[slots.long()] = lens

    def logits(self, engine, R):
        if R is None:
            raise RuntimeError("TransformerScorer needs the synchronous driver")
        if R == 0:
            return self._buf, N.VS_DTYPE_F32
        t = engine.t
        Lmax = engine.max_len
        phys = t["row_phys"][:R].long()
        slot = t["row_slot"][:R].long()
        ln = t["row_len"][:R].long()
        pos = ln - 1
        tok = t["hist"].view(-1, Lmax)[phys, pos].long()
        x = (self.emb[tok] + self.pos[pos])[:, None, :]  # [R, 1, d]
        Tk = int(ln.max())
        self_keep = (torch.arange(Tk, device=x.device)[None, :] < ln[:, None])[:, None, None, :]
        S = int(self.enc_len[slot].max())
        cross_keep = (torch.arange(S, device=x.device)[None, :] < self.enc_len[slot][:, None])[:, None, None, :]
        for li, L in enumerate(self.dec):
            q, k, v = (x @ L["qkv"].T).split(self.d, dim=-1)
            self.kv[2 * li, phys, pos] = k[:, 0]
            self.kv[2 * li + 1, phys, pos] = v[:, 0]
            K = self.kv[2 * li, phys, :Tk]
            Vv = self.kv[2 * li + 1, phys, :Tk]
            a = self._merge(self._attn(self._split(q), self._split(K), self._split(Vv), self_keep))
            x = F.layer_norm(x + a @ L["o"].T, (self.d,))
            cq = x @ L["cq"].T
            ck = self.enc_kv[slot, 2 * li, :S]
            cv = self.enc_kv[slot, 2 * li + 1, :S]
            a = self._merge(self._attn(self._split(cq), self._split(ck), self._split(cv), cross_keep))
            x = F.layer_norm(x + a @ L["co"].T, (self.d,))
            x = F.layer_norm(x + F.gelu(x @ L["f1"].T) @ L["f2"].T, (self.d,))
        lg = self._buf[:R]
        torch.matmul(x[:, 0], self.out.T, out=lg) if self.dtype == torch.float32 else lg.copy_(x[:, 0] @ self.out.T)
        lg.mul_(self.tau)
        src_len = t["slot_src_len"][slot].float()
        lg[:, self.vocab.eos] += self.eos_bias * ln.float() / src_len
        return self._buf, N.VS_DTYPE_F32

    def after_step(self, engine, R) -> None:
        # K4: apply K2's copy plan to every (layer, K|V) plane of the cache
        kv = self.kv
        es = kv.element_size()
        if self.record_logits:
            self.copies += int(engine.t["n_copy"].item())
        N.check(engine.lib.vs_rows_copy(kv.data_ptr(), kv.stride(0) * es, kv.shape[0], kv.stride(1) * es,
                                        kv.stride(2) * es, engine.t["copy_list"].data_ptr(),
                                        engine.t["n_copy"].data_ptr(), engine.max_copies, engine.stream_ptr),
                "vs_rows_copy")


class GraphedTransformerScorer(TransformerScorer):
    """WMT-shape decoder scorer (bf16, head_dim 64) for throughput runs.

    Same model as TransformerScorer (weights, post-LN layers, EOS bias), run
    as one CUDA graph per step-size bucket:

    * self-attention reads each row's prefix in place from the physical-row
      K/V cache and appends the new position in the same launch
      (vs_row_attention); cross-attention reads the slot's encoder states in
      place (no per-step gathers);
    * the step's row count lives on the device (status[VS_ST_R]); the graph
      for bucket Rb = roundup(R, 128) masks the padded rows (they write a
      dummy cache row), so shapes are static and every launch of the decoder
      step is a single graph replay;
    * tau is folded into W_out (logits in bf16, the K1 input dtype).

    K4 (after_step) and the encoder refill (on_admit) run outside the graph.
    """

    BUCKET = 128

    def __init__(self, vocab: Vocabulary, *, d: int = 1024, heads: int = 16, layers: int = 6,
                 enc_layers: int = 6, ffn: int = 4096, max_src: int = 256, seed: int = 0,
                 tau: float = 4.0, eos_bias: float = 4.0, device=None, use_graphs: bool = True,
                 fused_head: bool = False):
        if d % heads or d // heads != 64:
            raise ValueError("GraphedTransformerScorer needs head_dim 64")
        if max_src > 256:  # vs_row_attention_grouped stages <= 256 encoder positions per slot
            raise ValueError("GraphedTransformerScorer needs max_src <= 256")
        super().__init__(vocab, d=d, heads=heads, layers=layers, enc_layers=enc_layers, ffn=ffn,
                         max_src=max_src, seed=seed, tau=tau, eos_bias=eos_bias, dtype=torch.bfloat16,
                         device=device)
        self.out_s = (self.out.float() * tau).to(torch.bfloat16).contiguous()
        self.use_graphs = use_graphs
        self.fused_head = fused_head  # K5: tcgen05 vocab projection with K1 fused into the epilogue
        self.graphs = {}

    def _project(self, h):
        return (h @ self.out_s.T).float()

    def fork(self) -> "GraphedTransformerScorer":
        """Same weights (shared tensors), separate caches/graphs: a scorer for
        another engine running a concurrent batch."""
        import copy

        other = copy.copy(self)
        other._bound = None
        other.graphs = {}
        other.pool = None
        return other

    def bind(self, engine) -> None:
        n, k, Lmax = engine.n, engine.k, engine.max_len
        if Lmax > self.pos.shape[0]:
            raise ValueError("max_len exceeds the decoder's positions")
        dev, d = engine.device, self.d
        key = (id(engine), n, k, Lmax, engine.capacity)
        if getattr(self, "_bound", None) != key:  # (re)allocate; graphs capture these buffers
            self.engine = engine
            rows = n * k + 1  # + one dummy row for padded step rows
            self.dummy = n * k
            self.kv = torch.empty(self.nl, 2, rows, Lmax, d, device=dev, dtype=torch.bfloat16)
            self.enc_kv = torch.zeros(self.nl, 2, n, self.max_src, d, device=dev, dtype=torch.bfloat16)
            self.enc_len = torch.zeros(n, dtype=torch.int32, device=dev)
            ld = (self.vocab.size + 7) // 8 * 8
            self.lg = torch.empty(engine.capacity, ld, device=dev, dtype=torch.bfloat16)
            if self.fused_head:
                nb = int(engine.lib.vs_proj_lse_topm_ws_bytes(engine.capacity, self.vocab.size))
                self.k5_ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)
            self.graphs = {}
            self.pool = None
            self._bound = key
        self.enc_len.zero_()
        self._corpus_off = engine.t["src_off"].cpu().numpy()
        self._corpus_tok = engine.t["src_tok"].cpu().numpy()

    def on_admit(self, engine, status) -> None:
        n = engine.n
        a0, na = int(status[N.ST_ADMIT0]), int(status[N.ST_NADMIT])
        slots = torch.tensor(status[N.ST_HDR + 3 * n:N.ST_HDR + 3 * n + na].astype("int64"),
                             device=engine.device)
        srcs = [self._corpus_tok[self._corpus_off[i]:self._corpus_off[i + 1]] for i in range(a0, a0 + na)]
        lens = torch.tensor([len(s_) for s_ in srcs], device=engine.device)
        S = int(lens.max())
        if S > self.max_src:
            raise ValueError("source longer than the encoder's max_src")
        pad = torch.zeros(na, S, dtype=torch.long)
        for i, s_ in enumerate(srcs):
            pad[i, : len(s_)] = torch.from_numpy(s_.astype("int64"))
        cross = self.encode_sources(pad.to(engine.device), lens)
        # K4, encoder half: each admitted source's cross-attention K/V rows into its slot
        slots32 = slots.to(torch.int32)
        es = self.enc_kv.element_size()
        for li, (ck, cv) in enumerate(cross):
            for plane, src in ((0, ck), (1, cv)):
                src = src.contiguous()
                dst = self.enc_kv[li, plane]
                N.check(engine.lib.vs_scatter_rows(dst.data_ptr(), dst.stride(0) * es, src.data_ptr(),
                                                   src.stride(0) * es, S * self.d * es, slots32.data_ptr(),
                                                   None, na, engine.stream_ptr), "vs_scatter_rows")
        self.enc_len[slots] = lens.to(torch.int32)

    def _ln(self, x):
        """LayerNorm of the [rows, d] bf16 activations (vs_layer_norm_bf16)."""
        y = torch.empty_like(x)
        N.check(self.engine.lib.vs_layer_norm_bf16(x.data_ptr(), x.stride(0), y.data_ptr(), y.stride(0), x.shape[0],
                                                   self.d, 1e-5, torch.cuda.current_stream(self.device).cuda_stream),
                "vs_layer_norm_bf16")
        return y

    def _row_attn(self, q, kc, vc, idx, lens, knew, vnew, out):
        lib = self.engine.lib
        R = q.shape[0]
        N.check(lib.vs_row_attention(
            q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(), kc.stride(0), kc.stride(1),
            idx.data_ptr(), lens.data_ptr(), knew.data_ptr() if knew is not None else None,
            vnew.data_ptr() if vnew is not None else None, knew.stride(0) if knew is not None else 0,
            out.data_ptr(), out.stride(0), self.h, 64, 1.0 / 8.0, R, None, R,
            torch.cuda.current_stream(self.device).cuda_stream), "vs_row_attention")

    def _row_attn_grouped(self, q, kc, vc, idx, lens, out):
        """Cross-attention: the rows of one selected beam share the slot's encoder
        states (groups = engine sel_off / status NSEL; padded rows are not in any
        group and keep their self-attention output, finite and unused)."""
        eng = self.engine
        N.check(eng.lib.vs_row_attention_grouped(
            q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(), kc.stride(0), kc.stride(1),
            idx.data_ptr(), lens.data_ptr(), eng.t["sel_off"].data_ptr(), eng.status_ptr(N.ST_NSEL), eng.n,
            out.data_ptr(), out.stride(0), self.h, 64, 1.0 / 8.0,
            torch.cuda.current_stream(self.device).cuda_stream), "vs_row_attention_grouped")

    def _body(self, Rb: int):
        eng, t, d = self.engine, self.engine.t, self.d
        Lmax = eng.max_len
        R = t["status"][N.ST_R]
        valid = torch.arange(Rb, device=self.device, dtype=torch.int32) < R
        phys = t["row_phys"][:Rb]
        phys_kv = torch.where(valid, phys, self.dummy).to(torch.int32)
        slot = torch.where(valid, t["row_slot"][:Rb], 0).to(torch.int32)
        ln = torch.where(valid, t["row_len"][:Rb], 1).to(torch.int32)
        pos = (ln - 1).long()
        tok = t["hist"].view(-1, Lmax)[torch.where(valid, phys, 0).long(), pos].long()
        x = self.emb[tok] + self.pos[pos]
        enc_len = self.enc_len[slot.long()]
        att = torch.empty(Rb, d, device=self.device, dtype=torch.bfloat16)
        for li, L in enumerate(self.dec):
            qkv = x @ L["qkv"].T
            self._row_attn(qkv[:, :d], self.kv[li, 0], self.kv[li, 1], phys_kv, ln, qkv[:, d:2 * d],
                       qkv[:, 2 * d:], att)
            # residual adds in the GEMM epilogue (addmm: one rounding, no separate add kernel)
            x = self._ln(torch.addmm(x, att, L["o"].T))
            cq = x @ L["cq"].T
            self._row_attn_grouped(cq, self.enc_kv[li, 0], self.enc_kv[li, 1], slot, enc_len, att)
            x = self._ln(torch.addmm(x, att, L["co"].T))
            x = self._ln(torch.addmm(x, F.gelu(x @ L["f1"].T), L["f2"].T))
        lg = self.lg[:Rb, : self.vocab.size]
        eos = self.vocab.eos
        src_len = t["slot_src_len"][slot.long()].float()
        if self.fused_head:  # K5: projection + EOS bias + K1 in two launches
            eos_add = (self.eos_bias * ln.float() / src_len).contiguous()
            x = x.contiguous()
            N.check(eng.lib.vs_proj_lse_topm(
                x.data_ptr(), x.stride(0), self.out_s.data_ptr(), self.out_s.stride(0), Rb, None, Rb, d,
                self.vocab.size, eng.m_rows, eos, eos_add.data_ptr(), self.lg.data_ptr(), self.lg.stride(0),
                t["top_tok"].data_ptr(), t["top_logp"].data_ptr(), t["row_lse"].data_ptr(),
                t["fallbacks"].data_ptr(), self.k5_ws.data_ptr(), self.k5_ws.numel(),
                torch.cuda.current_stream(self.device).cuda_stream), "vs_proj_lse_topm")
            return lg
        torch.matmul(x, self.out_s.T, out=lg)
        lg[:, eos] = (lg[:, eos].float() + self.eos_bias * ln.float() / src_len).to(torch.bfloat16)
        return lg

    def logits(self, engine, R):
        if R is None:
            raise RuntimeError("GraphedTransformerScorer needs the synchronous driver")
        code = N.VS_K1_DONE if self.fused_head else N.VS_DTYPE_BF16
        if R == 0:
            return self.lg, N.VS_DTYPE_BF16
        Rb = min((R + self.BUCKET - 1) // self.BUCKET * self.BUCKET, engine.capacity)
        if not self.use_graphs:
            self._body(Rb)
            return self.lg, code
        g = self.graphs.get(Rb)
        if g is None:
            s = torch.cuda.Stream(self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(s):
                self._body(Rb)  # warm-up (idempotent: same rows, same writes)
            torch.cuda.current_stream(self.device).wait_stream(s)
            g = torch.cuda.CUDAGraph()
            if self.pool is None:
                self.pool = torch.cuda.graph_pool_handle()
            with torch.cuda.graph(g, pool=self.pool, capture_error_mode="thread_local"):
                self._body(Rb)
            self.graphs[Rb] = g
        g.replay()
        return self.lg, code

    def after_step(self, engine, R) -> None:
        kv = self.kv.view(self.nl * 2, *self.kv.shape[2:])
        es = kv.element_size()
        N.check(engine.lib.vs_rows_copy(kv.data_ptr(), kv.stride(0) * es, kv.shape[0], kv.stride(1) * es,
                                        kv.stride(2) * es, engine.t["copy_list"].data_ptr(),
                                        engine.t["n_copy"].data_ptr(), engine.max_copies, engine.stream_ptr),
                "vs_rows_copy")


class LSTMScorer:
    """BASELINE.json configs[2]: the lightweight LSTM encoder-decoder parsing
    shape (Dong & Lapata 2016 style): a 1-layer LSTM
    encoder over the source, a 1-layer LSTM decoder cell whose state is
    carried per PHYSICAL row, Luong dot attention over the slot's encoder
    states (4 heads of 64 on the tensor-core grouped kernel: the rows of a
    beam share their slot's states), h_att = tanh(W_c [h; ctx]) and logits
    tau * h_att W_out^T plus the EOS bias eos_bias*len/src_len (the structure
    of bb/model.py:215).  Random init (seeded), bf16 GEMM operands, fp32 cell
    state and nonlinearities.

    Per-row state (h, c) is a fixed-size record: extra children take a copy
    of their parent's (K4 vs_rows_copy in fixed-size mode), first children
    inherit the row.  A row of a freshly admitted beam (length 1) starts from
    its slot's encoder final state.  The step is one CUDA graph per row
    bucket (R from device memory, padded rows write a dummy row); the
    encoder runs at admission (cuDNN) and its states are placed by K4's
    vs_scatter_rows."""

    host_sync = True
    BUCKET = 128
    HEADS, DH = 4, 64

    def __init__(self, vocab: Vocabulary, *, emb: int = 128, hidden: int = 256, max_src: int = 128,
                 seed: int = 0, tau: float = 4.0, eos_bias: float = 4.0, device=None, use_graphs: bool = True):
        if hidden != self.HEADS * self.DH:
            raise ValueError(f"LSTMScorer attention needs hidden = {self.HEADS * self.DH}")
        if max_src > 256:
            raise ValueError("LSTMScorer needs max_src <= 256 (grouped attention staging)")
        self.vocab, self.E, self.H, self.max_src = vocab, emb, hidden, max_src
        self.tau, self.eos_bias, self.use_graphs = float(tau), float(eos_bias), use_graphs
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        g = torch.Generator(device="cpu").manual_seed(seed)
        V, E, H = vocab.size, emb, hidden

        def w(*shape, std=None):
            std = std if std is not None else 1.0 / math.sqrt(shape[-1])
            return torch.randn(*shape, generator=g) * std

        self.params = {
            "emb": w(V, E, std=1.0),
            "enc_ih": w(4 * H, E), "enc_hh": w(4 * H, H), "enc_b": w(4 * H, std=0.1),
            "dec_ih": w(4 * H, E), "dec_hh": w(4 * H, H), "dec_b": w(4 * H, std=0.1),
            "wc": w(H, 2 * H), "out": w(V, H),
        }
        p = {k: v.to(self.device) for k, v in self.params.items()}
        bf = torch.bfloat16
        self.emb = p["emb"].to(bf)
        self.w_cell = torch.cat([p["dec_ih"], p["dec_hh"]], 1).to(bf).contiguous()  # [4H, E+H]
        self.b_cell = p["dec_b"].float()
        self.wc = p["wc"].to(bf).contiguous()
        self.out_s = (p["out"] * tau).to(bf).contiguous()  # tau folded, bf16 logits (K1 input)
        self.encoder = torch.nn.LSTM(E, H, batch_first=True).to(self.device)
        with torch.no_grad():
            self.encoder.weight_ih_l0.copy_(p["enc_ih"])
            self.encoder.weight_hh_l0.copy_(p["enc_hh"])
            self.encoder.bias_ih_l0.copy_(p["enc_b"])
            self.encoder.bias_hh_l0.zero_()
        self.graphs, self.pool, self._bound = {}, None, None

    graph_safe = False

    def fork(self) -> "LSTMScorer":
        import copy

        other = copy.copy(self)
        other.graphs, other.pool, other._bound = {}, None, None
        return other

    # ------------------------------------------------------------------ model
    def encode_sources(self, src: torch.Tensor, lens: torch.Tensor):
        """src [B, S] (padded), lens [B] -> (enc_out [B, S, H] bf16, h0, c0 [B, H] fp32)."""
        x = self.emb[src].float()
        packed = torch.nn.utils.rnn.pack_padded_sequence(x, lens.cpu(), batch_first=True, enforce_sorted=False)
        with torch.no_grad():
            out, (h, c) = self.encoder(packed)
        out, _ = torch.nn.utils.rnn.pad_packed_sequence(out, batch_first=True, total_length=src.shape[1])
        return out.to(torch.bfloat16), h[0], c[0]

    def _cell(self, tok, h, c):
        gates = (torch.cat([self.emb[tok], h.to(torch.bfloat16)], 1) @ self.w_cell.T).float() + self.b_cell
        i, f, gg, o = gates.chunk(4, dim=1)
        c2 = torch.sigmoid(f) * c + torch.sigmoid(i) * torch.tanh(gg)
        h2 = torch.sigmoid(o) * torch.tanh(c2)
        return h2, c2

    def _head(self, h, ctx, ln, src_len):
        hb = torch.tanh((torch.cat([h.to(torch.bfloat16), ctx], 1) @ self.wc.T).float()).to(torch.bfloat16)
        lg = hb @ self.out_s.T
        eos = self.vocab.eos
        lg[:, eos] = (lg[:, eos].float() + self.eos_bias * ln.float() / src_len).to(torch.bfloat16)
        return lg

    def full_forward(self, src_tokens, prefix):
        """Cache-free logits of the last position of `prefix` (tests)."""
        dev = self.device
        src = torch.tensor([list(src_tokens)], device=dev)
        enc, h, c = self.encode_sources(src, torch.tensor([len(src_tokens)]))
        for t in prefix:
            h, c = self._cell(torch.tensor([t], device=dev), h, c)
        q = h.to(torch.bfloat16).view(1, self.HEADS, self.DH).float()
        k = enc[0].float().view(-1, self.HEADS, self.DH)
        a = torch.softmax(torch.einsum("hd,shd->hs", q[0], k) / 8.0, dim=-1)
        ctx = torch.einsum("hs,shd->hd", a, k).reshape(1, -1).to(torch.bfloat16)
        return self._head(h, ctx, torch.tensor([len(prefix)], device=dev),
                          torch.tensor([float(len(src_tokens))], device=dev))[0].float()

    # --------------------------------------------------------- engine protocol
    def bind(self, engine) -> None:
        n, k, dev = engine.n, engine.k, engine.device
        key = (id(engine), n, k, engine.capacity)
        if self._bound != key:  # graphs capture these buffers
            self.engine = engine
            self.dummy = n * k
            self.state = torch.zeros(n * k + 1, 2, self.H, device=dev, dtype=torch.float32)
            self.enc = torch.zeros(n, self.max_src, self.H, device=dev, dtype=torch.bfloat16)
            self.enc_hc = torch.zeros(n, 2, self.H, device=dev, dtype=torch.float32)
            self.enc_len = torch.zeros(n, dtype=torch.int32, device=dev)
            ld = (self.vocab.size + 7) // 8 * 8
            self.lg = torch.empty(engine.capacity, ld, device=dev, dtype=torch.bfloat16)
            self.graphs, self.pool, self._bound = {}, None, key
        self.enc_len.zero_()
        self._corpus_off = engine.t["src_off"].cpu().numpy()
        self._corpus_tok = engine.t["src_tok"].cpu().numpy()

    def on_admit(self, engine, status) -> None:
        n = engine.n
        a0, na = int(status[N.ST_ADMIT0]), int(status[N.ST_NADMIT])
        slots = torch.tensor(status[N.ST_HDR + 3 * n:N.ST_HDR + 3 * n + na].astype("int32"), device=engine.device)
        srcs = [self._corpus_tok[self._corpus_off[i]:self._corpus_off[i + 1]] for i in range(a0, a0 + na)]
        lens = torch.tensor([len(s_) for s_ in srcs])
        S = int(lens.max())
        if S > self.max_src:
            raise ValueError("source longer than the encoder's max_src")
        pad = torch.zeros(na, S, dtype=torch.long)
        for i, s_ in enumerate(srcs):
            pad[i, : len(s_)] = torch.from_numpy(s_.astype("int64"))
        out, h, c = self.encode_sources(pad.to(engine.device), lens)
        hc = torch.stack([h, c], 1).contiguous()
        lib, st = engine.lib, engine.stream_ptr
        # K4, encoder half: each admitted source's states into its slot
        N.check(lib.vs_scatter_rows(self.enc.data_ptr(), self.enc.stride(0) * 2, out.data_ptr(), out.stride(0) * 2,
                                    S * self.H * 2, slots.data_ptr(), None, na, st), "vs_scatter_rows")
        N.check(lib.vs_scatter_rows(self.enc_hc.data_ptr(), self.enc_hc.stride(0) * 4, hc.data_ptr(),
                                    hc.stride(0) * 4, hc.stride(0) * 4, slots.data_ptr(), None, na, st),
                "vs_scatter_rows")
        self.enc_len[slots.long()] = lens.to(engine.device, torch.int32)

    def _body(self, Rb: int):
        eng, t = self.engine, self.engine.t
        Lmax = eng.max_len
        R = t["status"][N.ST_R]
        valid = torch.arange(Rb, device=self.device, dtype=torch.int32) < R
        phys = torch.where(valid, t["row_phys"][:Rb], 0).long()
        slot = torch.where(valid, t["row_slot"][:Rb], 0).to(torch.int32)
        ln = torch.where(valid, t["row_len"][:Rb], 1)
        tok = t["hist"].view(-1, Lmax)[phys, (ln - 1).long()].long()
        fresh = (ln == 1)[:, None]
        prev = torch.where(fresh[:, :, None], self.enc_hc[slot.long()], self.state[phys])
        h, c = self._cell(tok, prev[:, 0], prev[:, 1])
        self.state[torch.where(valid, phys, self.dummy)] = torch.stack([h, c], 1)
        q = h.to(torch.bfloat16).contiguous()
        ctx = torch.empty(Rb, self.H, device=self.device, dtype=torch.bfloat16)
        enc_len = self.enc_len[slot.long()]
        N.check(eng.lib.vs_row_attention_grouped(
            q.data_ptr(), q.stride(0), self.enc.data_ptr(), self.enc.data_ptr(), self.enc.stride(0),
            self.enc.stride(1), slot.data_ptr(), enc_len.data_ptr(), t["sel_off"].data_ptr(),
            eng.status_ptr(N.ST_NSEL), eng.n, ctx.data_ptr(), ctx.stride(0), self.HEADS, self.DH, 1.0 / 8.0,
            torch.cuda.current_stream(self.device).cuda_stream), "vs_row_attention_grouped")
        src_len = t["slot_src_len"][slot.long()].float()
        self.lg[:Rb, : self.vocab.size] = self._head(h, ctx, ln, src_len)

    def logits(self, engine, R):
        if R is None:
            raise RuntimeError("LSTMScorer needs the synchronous driver")
        if R == 0:
            return self.lg, N.VS_DTYPE_BF16
        Rb = min((R + self.BUCKET - 1) // self.BUCKET * self.BUCKET, engine.capacity)
        if not self.use_graphs:
            self._body(Rb)
            return self.lg, N.VS_DTYPE_BF16
        g = self.graphs.get(Rb)
        if g is None:
            saved = self.state.clone()
            s = torch.cuda.Stream(self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(s):
                self._body(Rb)  # warm-up
            torch.cuda.current_stream(self.device).wait_stream(s)
            self.state.copy_(saved)  # the warm-up advanced the rows' state once
            g = torch.cuda.CUDAGraph()
            if self.pool is None:
                self.pool = torch.cuda.graph_pool_handle()
            with torch.cuda.graph(g, pool=self.pool, capture_error_mode="thread_local"):
                self._body(Rb)
            self.state.copy_(saved)
            self.graphs[Rb] = g
        g.replay()
        return self.lg, N.VS_DTYPE_BF16

    def after_step(self, engine, R) -> None:
        # K4 in fixed-size mode: each planned copy moves the parent's whole (h, c) record
        st = self.state
        N.check(engine.lib.vs_rows_copy(st.data_ptr(), 0, 1, st.stride(0) * 4, -(st.stride(0) * 4),
                                        engine.t["copy_list"].data_ptr(), engine.t["n_copy"].data_ptr(),
                                        engine.max_copies, engine.stream_ptr), "vs_rows_copy")
