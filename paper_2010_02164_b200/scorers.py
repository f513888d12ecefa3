"""Scorer plug-ins for the device engine.

The reference plug-in is the per-candidate ``Scorer`` protocol
(bb/model.py:78-87: ``vocab``, ``encode(tokens, input_id)``,
``score_next(encoding, candidate) -> |V| log-probs``).  The device engine
scores a whole timestep at once, so its plug-in is the ``BatchedScorer``
protocol below: the scorer owns any per-row state (e.g. a KV cache laid out
by PHYSICAL row, include/varstream.h) and re-orders it from the engine's copy
plan after every step.

* ``DeviceHashScorer`` — synthetic device scorer (csrc/hash_scorer.cu):
  deterministic logits for every row without a host round trip; the search
  benchmark's stand-in for the decoder's vocab projection.
* ``HostScorerAdapter`` — wraps any reference-protocol Scorer so existing
  reference scorers drop in unchanged (rows computed on the host, uploaded as
  already-normalised log-probs).  Slow by construction; for parity and API
  compatibility.
"""

from __future__ import annotations

import ctypes as C
from typing import Protocol

import numpy as np
import torch

from . import _native as N
from .core import Candidate, Vocabulary
from .errors import DataError


class BatchedScorer(Protocol):
    vocab: Vocabulary

    def bind(self, engine) -> None:
        """Allocate per-row state for engine.n*engine.k physical rows."""

    def on_admit(self, engine, status) -> None:
        """Encode newly admitted sources (device status lists their slots)."""

    def logits(self, engine, R: int | None) -> tuple[torch.Tensor, int]:
        """Return ([rows, ld] logits on device, VS_DTYPE_* code).  R=None means
        the row count lives only on the device (status[VS_ST_R])."""

    def after_step(self, engine, R: int | None) -> None:
        """Apply engine's row copy plan (copy_list) to per-row state (K4)."""


class DeviceHashScorer:
    """Counter-hash logits (see csrc/hash_scorer.cu; CPU mirror in
    oracle/scorers.py:HashLogitsCPU).  logit = scale*u^power with u uniform in
    [0,1); EOS logit = eos_bias*len/src_len, like bb/model.py:215."""

    def __init__(self, vocab: Vocabulary, seed: int, *, scale: float = 8.0, power: int = 1,
                 eos_bias: float = 8.0, dtype: str = "bf16"):
        if dtype not in ("bf16", "f32"):
            raise ValueError("dtype must be 'bf16' or 'f32'")
        self.vocab, self.seed = vocab, int(seed)
        self.scale, self.power, self.eos_bias, self.dtype = float(scale), int(power), float(eos_bias), dtype
        self.code = N.VS_DTYPE_BF16 if dtype == "bf16" else N.VS_DTYPE_F32
        self._buf = None

    graph_safe = True  # launches device work only: the sync-free step can be a CUDA graph

    @property
    def signature(self) -> tuple:
        return ("hash", self.vocab.size, self.seed, self.scale, self.power, self.eos_bias, self.dtype)

    def graph_key(self) -> tuple:
        """What a captured step graph bakes in: parameters and buffer address."""
        return self.signature + (self._buf.data_ptr() if self._buf is not None else 0,)

    def fork(self) -> "DeviceHashScorer":
        """An identical scorer for another engine (concurrent batches)."""
        return DeviceHashScorer(self.vocab, self.seed, scale=self.scale, power=self.power,
                                eos_bias=self.eos_bias, dtype=self.dtype)

    def bind(self, engine) -> None:
        V = self.vocab.size
        ld = (V + 7) // 8 * 8  # 16-byte aligned rows
        tdt = torch.bfloat16 if self.dtype == "bf16" else torch.float32
        if self._buf is None or self._buf.shape[0] < engine.capacity or self._buf.device != engine.device:
            self._buf = torch.empty((engine.capacity, ld), dtype=tdt, device=engine.device)
        self.params = N.VsHashParams(seed=self.seed & ((1 << 64) - 1), scale=self.scale,
                                     eos_bias=self.eos_bias, power=self.power, dtype=self.code)

    def on_admit(self, engine, status) -> None:
        pass  # the logits kernel encodes admitted sources inline (rows of length 1)

    def logits(self, engine, R):
        grid = engine.capacity if R is None else R
        if grid > 0:
            N.check(engine.lib.vs_hash_logits(C.byref(engine.cfg), C.byref(engine.state),
                                              C.byref(self.params), self._buf.data_ptr(),
                                              self._buf.stride(0), grid, engine.stream_ptr),
                    "vs_hash_logits")
        return self._buf, self.code

    def after_step(self, engine, R) -> None:
        pass  # all per-row state of this scorer is the candidate hash (moved by K2)


class HostScorerAdapter:
    """Runs a reference-protocol Scorer (bb/model.py:78-87) inside the device
    engine: candidates of the step's rows are rebuilt on the host, score_next
    is called per row in beam order (bb/search.py:223-225) and the rows are
    uploaded as the scorer's own fp64 log-probs (bb/model.py:216-217): the
    device selects the top-M by exact fp64 row value and adds those values in
    fp64 (vs_row_topm_f64), so a reference scorer's decode is bit-identical to
    the reference's — tokens, scores, events."""

    def __init__(self, scorer, corpus=None):
        self.inner = scorer
        v = scorer.vocab
        self.vocab = Vocabulary(v.size, v.sos, v.eos) if not isinstance(v, Vocabulary) else v
        self.corpus = corpus
        self.enc = {}

    def bind(self, engine) -> None:
        self.enc = {}
        self._buf = torch.empty((engine.capacity, self.vocab.size), dtype=torch.float64,
                                device=engine.device)

    def on_admit(self, engine, status) -> None:
        n = engine.n
        a0, na = int(status[N.ST_ADMIT0]), int(status[N.ST_NADMIT])
        slots = status[N.ST_HDR + 3 * n:N.ST_HDR + 3 * n + na]
        for q in range(na):
            iid = a0 + q
            self.enc[int(slots[q])] = self.inner.encode(self.corpus[iid], input_id=iid)

    def logits(self, engine, R):
        if R is None:
            raise RuntimeError("HostScorerAdapter needs the host row count (synchronous driver)")
        if R == 0:
            return self._buf, N.VS_DTYPE_F64 | N.VS_ROWS_NORMALIZED
        t = engine.t
        slots = t["row_slot"][:R].cpu().numpy()
        cands = t["row_cand"][:R].cpu().numpy()
        phys = t["row_phys"][:R].cpu().numpy()
        lens = t["row_len"][:R].cpu().numpy()
        k, L = engine.k, engine.max_len
        hist = t["hist"].view(-1, L)[torch.from_numpy(phys).to(engine.device).long()].cpu().numpy()
        score = t["c_score"][(torch.from_numpy(slots * k + cands)).to(engine.device).long()].cpu().numpy()
        rows = np.empty((R, self.vocab.size), dtype=np.float64)
        for r in range(R):
            enc = self.enc[int(slots[r])]
            cand = Candidate(tuple(int(x) for x in hist[r, :lens[r]]), float(score[r]), False,
                             enc.input_id)
            row = self.inner.score_next(enc, cand)
            if len(row) != self.vocab.size:
                raise DataError(f"score row of length {len(row)} for vocabulary of size "
                                f"{self.vocab.size}")
            rows[r] = np.asarray(row, dtype=np.float64)
        self._buf[:R].copy_(torch.from_numpy(rows))
        return self._buf, N.VS_DTYPE_F64 | N.VS_ROWS_NORMALIZED

    def after_step(self, engine, R) -> None:
        pass


class LseRecorder:
    """Parity-mode wrapper (SURVEY.md §7 hard part 2): records, for every scored
    row, the kernel's lse keyed by (input_id, candidate tokens) so a CPU replay
    can rebuild the exact rows the search saw: float64(fp32(logit - lse)).
    Synchronous driver only (it reads the row list on the host each step)."""

    host_sync = True

    def __init__(self, inner, record_logits: bool = False):
        self.inner = inner
        self.vocab = inner.vocab
        self.table = {}
        self.logit_table = {} if record_logits else None
        self._keys = None
        self._logits = None

    def bind(self, engine) -> None:
        self.inner.bind(engine)

    def on_admit(self, engine, status) -> None:
        self.inner.on_admit(engine, status)

    def logits(self, engine, R):
        if R is None:
            raise RuntimeError("LseRecorder needs the synchronous driver")
        out = self.inner.logits(engine, R)
        t, L, k = engine.t, engine.max_len, engine.k
        if self.logit_table is not None and R:
            lg, code = out
            self._logits = lg[:R, : self.vocab.size].float().cpu().numpy()
        if R:
            phys = t["row_phys"][:R].long()
            hist = t["hist"].view(-1, L)[phys].cpu().numpy()
            lens = t["row_len"][:R].cpu().numpy()
            inputs = t["slot_input"][t["row_slot"][:R].long()].cpu().numpy()
            self._keys = [(int(inputs[r]), tuple(int(x) for x in hist[r, :lens[r]]))
                          for r in range(R)]
        else:
            self._keys = []
        return out

    def after_step(self, engine, R) -> None:
        lse = engine.t["row_lse"][:R].cpu().numpy() if R else []
        for i, (key, v) in enumerate(zip(self._keys, lse)):
            self.table[key] = np.float32(v)
            if self.logit_table is not None:
                self.logit_table[key] = self._logits[i].copy()
        self.inner.after_step(engine, R)
