"""CPU scorers for the oracle (TEST INFRASTRUCTURE).

* ``SeededHashScorerCPU`` restates the reference's synthetic scorer
  (bb/model.py:177-218: blake2b-keyed PCG64 logits, EOS logit
  ``eos_bias*len/input_len``, fp64 log-softmax).  It is only used to pin this
  oracle against outputs of the real reference (tests/golden).
* ``HashLogitsCPU`` is the bit-exact CPU mirror of the product's device
  synthetic scorer (paper_2010_02164_b200/csrc/hash_scorer.cu): a counter
  hash of (seed, source, candidate prefix, token) -> fp32 (optionally bf16)
  logits computed with IEEE-exact ops only, so CPU and GPU logits agree bit for
  bit.
* ``LseReplayScorer`` turns those logits into the rows the reference search
  would see given the kernel's per-row ``lse``: ``float64(fp32(logit - lse))``
  (SURVEY.md §7 hard part 2: the log-softmax contract).
"""

from __future__ import annotations

import hashlib
import math
import struct
from dataclasses import dataclass

import numpy as np

M64 = (1 << 64) - 1


@dataclass(frozen=True, slots=True)
class Encoding:
    """bb/model.py:34-45."""

    input_id: int
    tokens: tuple
    input_len: int
    seed: int = 0


def _check_input_tokens(tokens, vocab_size: int) -> tuple:
    """bb/model.py:90-102."""
    if len(tokens) == 0:
        raise ValueError("inputs must be nonempty")
    out = []
    for pos, t in enumerate(tokens):
        t = int(t)
        if not (0 <= t < vocab_size):
            raise ValueError(f"token {t} at position {pos} is outside the vocabulary "
                             f"(size {vocab_size})")
        out.append(t)
    return tuple(out)


class SeededHashScorerCPU:
    """Restatement of bb/model.py:177-218 (SeededHashScorer)."""

    def __init__(self, vocab_size: int, sos: int, eos: int, seed: int, eos_bias: float = 0.0):
        self.vocab_size, self.sos, self.eos = vocab_size, sos, eos
        self.seed = int(seed)
        self.eos_bias = float(eos_bias)
        self._key = struct.pack("<q", self.seed)

    def _digest(self, tag: bytes, tokens: tuple, extra: int = 0) -> int:  # :195-198
        payload = tag + struct.pack("<Q", extra) + struct.pack(f"<{len(tokens)}Q", *tokens)
        return int.from_bytes(hashlib.blake2b(payload, digest_size=8, key=self._key).digest(),
                              "little")

    def encode(self, tokens, input_id: int = 0) -> Encoding:  # :200-207
        checked = _check_input_tokens(tokens, self.vocab_size)
        return Encoding(input_id, checked, len(checked), self._digest(b"enc", checked))

    def score_next(self, enc: Encoding, cand):  # :209-218
        if cand.finalized:
            raise RuntimeError("scoring a finalized candidate")
        state = self._digest(b"dec", tuple(cand.tokens), extra=enc.seed)
        rng = np.random.Generator(np.random.PCG64(state))
        logits = rng.random(self.vocab_size)
        logits[self.eos] = self.eos_bias * len(cand.tokens) / enc.input_len
        peak = logits.max()
        return logits - (peak + math.log(np.exp(logits - peak).sum()))


# ------------------------------------------------------ device scorer mirror
def mix64(z: int) -> int:
    """splitmix64 finalizer (same constants as csrc/hash_scorer.cu)."""
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def source_seed(seed: int, tokens) -> int:
    h = mix64((seed ^ 0x9E3779B97F4A7C15) & M64)
    for t in tokens:
        h = mix64(h ^ ((int(t) + 0x632BE59BD9B4E019) & M64))
    return h


def prefix_init(src_seed: int, sos: int) -> int:
    return mix64((src_seed + (sos + 1) * 0xD6E8FEB86659FD93) & M64)


def prefix_step(h: int, token: int) -> int:
    return mix64(h ^ (((token + 1) * 0xD6E8FEB86659FD93) & M64))


def prefix_hash(src_seed: int, tokens) -> int:
    h = prefix_init(src_seed, int(tokens[0]))
    for t in tokens[1:]:
        h = prefix_step(h, int(t))
    return h


def fmix32_np(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint32)
    x ^= x >> np.uint32(16)
    x *= np.uint32(0x85EBCA6B)
    x ^= x >> np.uint32(13)
    x *= np.uint32(0xC2B2AE35)
    x ^= x >> np.uint32(16)
    return x


def f32_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """IEEE round-to-nearest-even fp32 -> bf16, returned widened to fp32
    (matches __float2bfloat16_rn for finite values)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


class HashLogitsCPU:
    """Bit-exact CPU mirror of the device synthetic scorer's logits.

    logit[v] = scale * u^power, u = (fmix32(key ^ v*0x9E3779B9) >> 8) * 2^-24
    (key folds the candidate's prefix hash); power=0 is the log-like mode
    logit = -scale * (e + f) for u' = u + 2^-24 = 2^e (1 + f) (a bit-cast log2,
    exponential upper tail like real LM logits); and
    logit[eos] = (eos_bias * len) / src_len, all fp32 round-to-nearest; in
    bf16 mode each logit is then rounded to bf16.  Mirrors the structure of
    bb/model.py:209-218 with an integer hash in place of blake2b+PCG64."""

    def __init__(self, vocab_size: int, sos: int, eos: int, seed: int, *, scale: float = 8.0,
                 power: int = 1, eos_bias: float = 8.0, dtype: str = "f32"):
        assert power in (0, 1, 2, 4)
        self.vocab_size, self.sos, self.eos = vocab_size, sos, eos
        self.seed, self.scale, self.power = int(seed), np.float32(scale), power
        self.eos_bias, self.dtype = np.float32(eos_bias), dtype
        self._v = np.arange(vocab_size, dtype=np.uint32) * np.uint32(0x9E3779B9)

    def encode(self, tokens, input_id: int = 0) -> Encoding:
        checked = tuple(int(t) for t in tokens)
        if not checked:
            raise ValueError("inputs must be nonempty")
        return Encoding(input_id, checked, len(checked), source_seed(self.seed, checked))

    def logits(self, enc: Encoding, tokens) -> np.ndarray:
        h = prefix_hash(enc.seed, tokens)
        key = np.uint32((h ^ (h >> 32)) & 0xFFFFFFFF)
        bits = fmix32_np(self._v ^ key)
        if self.power == 0:  # log-like: x = -scale * (e + f) with u = 2^e (1 + f)
            b = (bits >> np.uint32(8)) + np.uint32(1)
            u = b.astype(np.float32) * np.float32(2.0 ** -24)
            ub = u.view(np.uint32)
            e = (ub >> np.uint32(23)).astype(np.int32) - 127
            f = (ub & np.uint32(0x7FFFFF)).astype(np.float32) * np.float32(2.0 ** -23)
            x = (np.float32(-self.scale) * (e.astype(np.float32) + f)).astype(np.float32)
        else:
            u = (bits >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)
            if self.power >= 2:
                u = u * u
            if self.power >= 4:
                u = u * u
            x = (u * self.scale).astype(np.float32)
        x[self.eos] = (self.eos_bias * np.float32(len(tokens))) / np.float32(enc.input_len)
        if self.dtype == "bf16":
            x = f32_to_bf16_rne(x)
        return x

    def score_next(self, enc: Encoding, cand):
        """Standalone CPU rows (fp64 log-softmax of the fp32 logits, as the
        reference does).  GPU parity uses LseReplayScorer instead."""
        x = self.logits(enc, cand.tokens).astype(np.float64)
        peak = x.max()
        return x - (peak + math.log(np.exp(x - peak).sum()))


class LseReplayScorer:
    """Reference-protocol scorer whose rows are float64(fp32(logit - lse)),
    with lse exported by the kernel per (input_id, tokens)."""

    def __init__(self, base: HashLogitsCPU, lse_table: dict):
        self.base = base
        self.vocab_size, self.sos, self.eos = base.vocab_size, base.sos, base.eos
        self.lse = lse_table

    def encode(self, tokens, input_id: int = 0):
        return self.base.encode(tokens, input_id)

    def score_next(self, enc: Encoding, cand):
        x = self.base.logits(enc, cand.tokens)
        lse = np.float32(self.lse[(enc.input_id, tuple(cand.tokens))])
        return (x - lse).astype(np.float32).astype(np.float64)


class RowsScorer:
    """tests/support.py:238-250: replays pre-drawn rows in call order."""

    def __init__(self, vocab_size: int, sos: int, eos: int, rows):
        self.vocab_size, self.sos, self.eos = vocab_size, sos, eos
        self._rows = list(rows)

    def encode(self, tokens, input_id: int = 0):
        return Encoding(input_id, tuple(tokens), len(tokens))

    def score_next(self, enc, cand):
        return self._rows.pop(0)


class RecordedRowsScorer:
    """Replays rows recorded from a device scorer (logits + kernel lse per
    (input_id, tokens)): float64(fp32(logit - lse)).  Used for decoders whose
    logits the CPU cannot recompute bit-exactly."""

    def __init__(self, vocab_size: int, sos: int, eos: int, logits: dict, lse: dict):
        self.vocab_size, self.sos, self.eos = vocab_size, sos, eos
        self.logits, self.lse = logits, lse

    def encode(self, tokens, input_id: int = 0):
        return Encoding(input_id, tuple(int(t) for t in tokens), len(tokens))

    def score_next(self, enc, cand):
        key = (enc.input_id, tuple(cand.tokens))
        x = np.asarray(self.logits[key], dtype=np.float32)
        return (x - np.float32(self.lse[key])).astype(np.float32).astype(np.float64)


class TorchDecoderCPU:
    """Reference-protocol scorer (bb/model.py:78-87: ``encode``, stateless
    ``score_next``) for the WMT'19-shape decoder leg's CPU baseline: the
    random-init transformer of paper_2010_02164_b200/decoder.py rebuilt on the
    CPU from the same seeded generator sequence (identical bf16 weights, fp32
    compute), recomputing the whole prefix for every candidate as the
    reference's stateless scorer protocol does.  Rows are the fp64
    log-softmax of the logits (bb/model.py:216-217).  TEST/BASELINE
    INFRASTRUCTURE: only bench.py's cpu-baseline legs use it."""

    def __init__(self, vocab_size: int, sos: int, eos: int, *, d: int = 1024, heads: int = 16,
                 layers: int = 6, enc_layers: int = 6, ffn: int = 4096, seed: int = 0, tau: float = 6.0,
                 eos_bias: float = 20.0, weights: str = "bf16"):
        import torch

        self.torch = torch
        self.vocab_size, self.sos, self.eos = vocab_size, sos, eos
        self.d, self.h, self.tau, self.eos_bias = d, heads, tau, eos_bias
        g = torch.Generator(device="cpu").manual_seed(seed)
        rnd = (lambda t: t.to(torch.bfloat16).float()) if weights == "bf16" else (lambda t: t)

        def w(*shape, std=None):  # same draw order / scaling as decoder.TransformerScorer
            std = std if std is not None else 1.0 / math.sqrt(shape[-1])
            return rnd(torch.randn(*shape, generator=g) * std)

        V = vocab_size
        self.emb = w(V, d, std=1.0)
        self.pos = w(512, d, std=0.5)
        self.enc = [dict(qkv=w(3 * d, d), o=w(d, d), f1=w(ffn, d), f2=w(d, ffn)) for _ in range(enc_layers)]
        self.dec = [dict(qkv=w(3 * d, d), o=w(d, d), cq=w(d, d), ckv=w(2 * d, d), co=w(d, d),
                         f1=w(ffn, d), f2=w(d, ffn)) for _ in range(layers)]
        out = torch.randn(V, d, generator=g) * (1.0 / math.sqrt(d))
        if weights == "bf16":  # tau folded into the bf16 weight, as GraphedTransformerScorer does
            self.out_s = (out.to(torch.bfloat16).float() * tau).to(torch.bfloat16).float()
            self.post_tau = 1.0
        else:  # fp32 TransformerScorer: tau * (h @ W_out^T)
            self.out_s, self.post_tau = out, tau

    def _attn(self, q, k, v, mask):
        F = self.torch.nn.functional
        dh = self.d // self.h

        def split(x):
            B, T, _ = x.shape
            return x.view(B, T, self.h, dh).transpose(1, 2)

        s = (split(q) @ split(k).transpose(-1, -2)) / math.sqrt(dh)
        if mask is not None:
            s = s.masked_fill(~mask, float("-inf"))
        a = F.softmax(s, dim=-1) @ split(v)
        B, h, T, _ = a.shape
        return a.transpose(1, 2).reshape(B, T, h * dh)

    def encode(self, tokens, input_id: int = 0) -> Encoding:
        torch, F = self.torch, self.torch.nn.functional
        toks = _check_input_tokens(tokens, self.vocab_size)
        with torch.no_grad():
            x = (self.emb[list(toks)] + self.pos[: len(toks)])[None]
            for L in self.enc:
                q, k, v = (x @ L["qkv"].T).split(self.d, dim=-1)
                x = F.layer_norm(x + self._attn(q, k, v, None) @ L["o"].T, (self.d,))
                x = F.layer_norm(x + F.gelu(x @ L["f1"].T) @ L["f2"].T, (self.d,))
            cross = [(x @ L["ckv"].T).split(self.d, dim=-1) for L in self.dec]
        enc = Encoding(input_id, toks, len(toks))
        self._cross = getattr(self, "_cross", {})
        self._cross[(input_id, toks)] = cross
        return enc

    def score_next(self, enc: Encoding, cand):
        if getattr(self, "incremental", False):
            return self.score_batch(enc, [cand])[0]
        torch, F = self.torch, self.torch.nn.functional
        cross = self._cross[(enc.input_id, enc.tokens)]
        prefix = list(cand.tokens)
        T = len(prefix)
        with torch.no_grad():
            x = (self.emb[prefix] + self.pos[:T])[None]
            causal = torch.ones(T, T, dtype=torch.bool).tril()[None, None]
            for L, (ck, cv) in zip(self.dec, cross):
                q, k, v = (x @ L["qkv"].T).split(self.d, dim=-1)
                x = F.layer_norm(x + self._attn(q, k, v, causal) @ L["o"].T, (self.d,))
                x = F.layer_norm(x + self._attn(x @ L["cq"].T, ck, cv, None) @ L["co"].T, (self.d,))
                x = F.layer_norm(x + F.gelu(x @ L["f1"].T) @ L["f2"].T, (self.d,))
            lg = (x[0, -1] @ self.out_s.T)
            lg = (lg * self.post_tau if self.post_tau != 1.0 else lg).double()
        lg[self.eos] += self.eos_bias * T / enc.input_len
        peak = float(lg.max())
        return (lg - (peak + math.log(float(torch.exp(lg - peak).sum())))).numpy()


    def score_batch(self, enc: Encoding, cands):
        """Incremental mode: rows for several candidates of one beam (all of one
        length) in one batched pass per layer and one vocab GEMM, with each
        prefix's per-layer K/V cached by token tuple (a candidate's parent
        holds positions 0..T-2).  The model is unchanged; only the fp32
        evaluation order differs from whole-prefix recompute."""
        import collections

        torch, F = self.torch, self.torch.nn.functional
        if not hasattr(self, "_kv"):
            self._kv = collections.OrderedDict()
        if len({len(c.tokens) for c in cands}) != 1:
            return [r for c in cands for r in self.score_batch(enc, [c])]
        cross = self._cross[(enc.input_id, enc.tokens)]
        T = len(cands[0].tokens)
        parents = []
        for c in cands:
            key = (enc.input_id, tuple(c.tokens[:-1]))
            if T > 1 and key not in self._kv:  # not cached: build the prefix first

                class _P:
                    tokens = tuple(c.tokens[:-1])

                self.score_batch(enc, [_P])
            parents.append(self._kv[key] if T > 1 else None)
        d, B = self.d, len(cands)
        with torch.no_grad():
            x = (self.emb[[c.tokens[-1] for c in cands]] + self.pos[T - 1])[:, None]  # [B, 1, d]
            per_row = [[] for _ in range(B)]
            for li, (L, (ck, cv)) in enumerate(zip(self.dec, cross)):
                q, k, v = (x @ L["qkv"].T).split(d, dim=-1)
                if T > 1:
                    K = torch.cat([torch.stack([p[li][0] for p in parents]), k], 1)
                    Vv = torch.cat([torch.stack([p[li][1] for p in parents]), v], 1)
                else:
                    K, Vv = k, v
                for b in range(B):
                    per_row[b].append((K[b], Vv[b]))
                x = F.layer_norm(x + self._attn(q, K, Vv, None) @ L["o"].T, (d,))
                x = F.layer_norm(x + self._attn(x @ L["cq"].T, ck.expand(B, -1, -1), cv.expand(B, -1, -1), None)
                                 @ L["co"].T, (d,))
                x = F.layer_norm(x + F.gelu(x @ L["f1"].T) @ L["f2"].T, (d,))
            lg = x[:, 0] @ self.out_s.T
            lg = (lg * self.post_tau if self.post_tau != 1.0 else lg).double()
        for b, c in enumerate(cands):
            self._kv[(enc.input_id, tuple(c.tokens))] = per_row[b]
        while len(self._kv) > 512:
            self._kv.popitem(last=False)
        lg[:, self.eos] += self.eos_bias * T / enc.input_len
        peak = lg.max(dim=1, keepdim=True).values
        return list((lg - (peak + torch.log(torch.exp(lg - peak).sum(dim=1, keepdim=True)))).numpy())

class LSTMDecoderCPU:
    """Reference-protocol scorer (bb/model.py:78-87: ``encode``, stateless
    ``score_next``) for the configs[2] LSTM leg's CPU baseline: the random-init
    model of paper_2010_02164_b200/decoder.py:LSTMScorer rebuilt on the CPU
    from the same seeded generator sequence (the same bf16-rounded operands,
    fp32 compute), re-running the decoder cell over the whole prefix for every
    candidate as the reference's stateless protocol does.  Rows are the fp64
    log-softmax of the logits (bb/model.py:216-217).  TEST/BASELINE
    INFRASTRUCTURE: only tests/ and bench.py's cpu-baseline legs use it."""

    HEADS, DH = 4, 64

    def __init__(self, vocab_size: int, sos: int, eos: int, *, emb: int = 128, hidden: int = 256,
                 seed: int = 0, tau: float = 4.0, eos_bias: float = 4.0):
        import torch

        self.torch = torch
        self.vocab_size, self.sos, self.eos = vocab_size, sos, eos
        self.H, self.tau, self.eos_bias = hidden, tau, eos_bias
        g = torch.Generator(device="cpu").manual_seed(seed)
        V, E, H = vocab_size, emb, hidden

        def w(*shape, std=None):  # same draw order / scaling as decoder.LSTMScorer
            std = std if std is not None else 1.0 / math.sqrt(shape[-1])
            return torch.randn(*shape, generator=g) * std

        bf = lambda t: t.to(torch.bfloat16).float()  # noqa: E731
        p = {"emb": w(V, E, std=1.0), "enc_ih": w(4 * H, E), "enc_hh": w(4 * H, H), "enc_b": w(4 * H, std=0.1),
             "dec_ih": w(4 * H, E), "dec_hh": w(4 * H, H), "dec_b": w(4 * H, std=0.1), "wc": w(H, 2 * H),
             "out": w(V, H)}
        self.emb = bf(p["emb"])
        self.w_cell = bf(torch.cat([p["dec_ih"], p["dec_hh"]], 1))
        self.b_cell = p["dec_b"]
        self.wc = bf(p["wc"])
        self.out_s = bf(p["out"] * tau)
        self.encoder = torch.nn.LSTM(E, H, batch_first=True)
        with torch.no_grad():
            self.encoder.weight_ih_l0.copy_(p["enc_ih"])
            self.encoder.weight_hh_l0.copy_(p["enc_hh"])
            self.encoder.bias_ih_l0.copy_(p["enc_b"])
            self.encoder.bias_hh_l0.zero_()
        self._enc = {}

    def encode(self, tokens, input_id: int = 0) -> Encoding:
        torch = self.torch
        toks = _check_input_tokens(tokens, self.vocab_size)
        with torch.no_grad():
            out, (h, c) = self.encoder(self.emb[list(toks)][None])
        self._enc[(input_id, toks)] = (out[0].to(torch.bfloat16).float(), h[0, 0], c[0, 0])
        return Encoding(input_id, toks, len(toks))

    def score_next(self, enc: Encoding, cand):
        torch = self.torch
        out, h, c = self._enc[(enc.input_id, enc.tokens)]
        bf = lambda t: t.to(torch.bfloat16).float()  # noqa: E731
        with torch.no_grad():
            for t in cand.tokens:
                gates = torch.cat([self.emb[t], bf(h)]) @ self.w_cell.T + self.b_cell
                i, f, gg, o = gates.chunk(4)
                c = torch.sigmoid(f) * c + torch.sigmoid(i) * torch.tanh(gg)
                h = torch.sigmoid(o) * torch.tanh(c)
            q = bf(h).view(self.HEADS, self.DH)
            k = out.view(-1, self.HEADS, self.DH)
            a = torch.softmax(torch.einsum("hd,shd->hs", q, k) / 8.0, dim=-1)
            ctx = bf(torch.einsum("hs,shd->hd", a, k).reshape(-1))
            hb = bf(torch.tanh(torch.cat([bf(h), ctx]) @ self.wc.T))
            lg = (hb @ self.out_s.T).double()
        lg[self.eos] += self.eos_bias * len(cand.tokens) / enc.input_len
        peak = float(lg.max())
        return (lg - (peak + math.log(float(torch.exp(lg - peak).sum())))).numpy()
