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
        lg = (x[0, -1] @ self.out.T).float() * self.tau
        lg[self.vocab.eos] += self.eos_bias * T / len(src_tokens)
        return lg

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
                                        engine.t["n_copy"].data_ptr(), engine.capacity, engine.stream_ptr),
                "vs_rows_copy")
