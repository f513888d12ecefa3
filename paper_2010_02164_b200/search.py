"""Per-beam and per-row entry points on the device (drop-ins for bb/search.py).

``expand_beam(beam, score_rows, config, vocab)`` has the signature and
semantics of bb/search.py:76-103 (deferred policy) but runs K1 + K2 on the
GPU; ``row_lse_topm`` exposes K1 alone (bb/model.py:216-217 +
bb/search.py:69) for batched use.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .core import Beam, Candidate, DecodeConfig, Vocabulary
from .engine import SearchEngine
from .errors import InvariantViolation


_WS: dict = {}


def k1_workspace(R_grid: int, V: int, code: int, device) -> torch.Tensor:
    """Zeroed K1 workspace (per-row counters return to zero after every
    launch, so one allocation serves every later call with the same V and
    dtype on the device; its layout depends on V and dtype only)."""
    lib = N.load_library()
    nbytes = int(lib.vs_row_lse_topm_ws_bytes(R_grid, V, code))
    key = (str(device), V, code & ~N.VS_ROWS_NORMALIZED)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def row_lse_topm(logits: torch.Tensor, M: int, *, normalized: bool = False, legacy: bool = False,
                 kernel: str = "auto"):
    """K1 over a [R, V] device tensor (fp32 or bf16; rows may be strided).
    Returns (tokens int32 [R, M], logp fp32 [R, M], lse fp32 [R], fallbacks).
    `kernel`: "auto" (library dispatch), "split" (TMA split-row kernel when
    the rows qualify) or "warp" (warp-per-row kernel); `legacy` calls the
    workspace-free entry point (always the warp-per-row kernel)."""
    if logits.dim() != 2 or logits.stride(1) != 1:
        raise ValueError("logits must be a row-major [R, V] tensor")
    R, V = logits.shape
    code = {torch.float32: N.VS_DTYPE_F32, torch.bfloat16: N.VS_DTYPE_BF16}[logits.dtype]
    if normalized:
        code |= N.VS_ROWS_NORMALIZED
    pin = {"auto": 0, "split": N.VS_K1_SPLIT, "warp": N.VS_K1_WARP}[kernel]
    dev = logits.device
    tok = torch.empty((R, M), dtype=torch.int32, device=dev)
    lp = torch.empty((R, M), dtype=torch.float32, device=dev)
    lse = torch.empty((R,), dtype=torch.float32, device=dev)
    fb = torch.zeros((1,), dtype=torch.int32, device=dev)
    lib = N.load_library()
    stream = torch.cuda.current_stream(dev).cuda_stream
    if legacy:
        N.check(lib.vs_row_lse_topm(logits.data_ptr(), code, logits.stride(0), V, M, R, None, R,
                                    tok.data_ptr(), lp.data_ptr(), lse.data_ptr(), fb.data_ptr(),
                                    stream), "vs_row_lse_topm")
    else:
        ws = k1_workspace(R, V, code, dev)
        N.check(lib.vs_row_lse_topm_ws(logits.data_ptr(), code | pin, logits.stride(0), V, M, R, None, R,
                                       tok.data_ptr(), lp.data_ptr(), lse.data_ptr(), fb.data_ptr(),
                                       ws.data_ptr(), ws.numel(), stream), "vs_row_lse_topm_ws")
    return tok, lp, lse, fb


def proj_lse_topm(h: torch.Tensor, w: torch.Tensor, M: int, *, eos: int = -1, eos_add=None):
    """K5 (tcgen05 vocab projection + fused K1): logits = bf16(h @ w^T) with the
    EOS bias, and K1's outputs on them.  h bf16 [R, K], w bf16 [V, K].
    Returns (tokens [R, M], logp [R, M], lse [R], fallbacks, logits [R, V])."""
    if h.dtype != torch.bfloat16 or w.dtype != torch.bfloat16 or h.shape[1] != w.shape[1]:
        raise ValueError("h [R, K] and w [V, K] must be bf16 with the same K")
    R, K = h.shape
    V = w.shape[0]
    dev = h.device
    tok = torch.empty((R, M), dtype=torch.int32, device=dev)
    lp = torch.empty((R, M), dtype=torch.float32, device=dev)
    lse = torch.empty((R,), dtype=torch.float32, device=dev)
    fb = torch.zeros((1,), dtype=torch.int32, device=dev)
    ld = (V + 7) // 8 * 8
    lg = torch.empty((R, ld), dtype=torch.bfloat16, device=dev)
    lib = N.load_library()
    ws = torch.empty(max(int(lib.vs_proj_lse_topm_ws_bytes(R, V)), 256), dtype=torch.uint8, device=dev)
    ea = eos_add.float().contiguous() if eos_add is not None else None
    N.check(lib.vs_proj_lse_topm(h.data_ptr(), h.stride(0), w.data_ptr(), w.stride(0), R, None, R, K, V, M, eos,
                                 ea.data_ptr() if ea is not None else None,
                                 lg.data_ptr(), ld, tok.data_ptr(), lp.data_ptr(),
                                 lse.data_ptr(), fb.data_ptr(), ws.data_ptr(), ws.numel(),
                                 torch.cuda.current_stream(dev).cuda_stream), "vs_proj_lse_topm")
    return tok, lp, lse, fb, lg[:, :V]


def _load_beam(eng: SearchEngine, beam: Beam) -> int:
    """Write one beam into slot 0 of a 1-slot engine; returns its active width."""
    k, L = eng.k, eng.max_len
    w = len(beam.candidates)
    t = eng.t
    t["slot_input"][0] = 0
    t["slot_lt"][0] = beam.l_t
    t["slot_emitted"][0] = beam.emitted
    t["slot_width"][0] = w
    nact = beam.active_width()
    t["slot_active"][0] = nact
    t["slot_flags"][0] = 1
    hist = np.zeros((k, L), dtype=np.int32)
    for j, c in enumerate(beam.candidates):
        hist[j, : len(c.tokens)] = c.tokens
    t["hist"].view(k, L).copy_(torch.from_numpy(hist))
    t["c_score"][:w] = torch.tensor([c.score for c in beam.candidates], dtype=torch.float64)
    t["c_len"][:w] = torch.tensor([len(c.tokens) for c in beam.candidates], dtype=torch.int32)
    t["c_row"][:w] = torch.arange(w, dtype=torch.int32)
    t["c_fin"][:w] = torch.tensor([int(c.finalized) for c in beam.candidates], dtype=torch.uint8)
    st = np.zeros(N.status_ints(1), dtype=np.int32)
    st[N.ST_R], st[N.ST_NSEL] = nact, 1
    t["status"].copy_(torch.from_numpy(st))
    t["sel"][0] = 0
    t["sel_off"][:2] = torch.tensor([0, nact], dtype=torch.int32)
    t["n_copy"].zero_()
    return nact


def expand_beam(beam: Beam, score_rows, config: DecodeConfig, vocab: Vocabulary,
                *, drain: bool = False):
    """Device expand_beam (bb/search.py:76-103).  Rows are per-active-candidate
    log-prob vectors in beam order; they are rounded to fp32 on upload (the
    kernel contract: logp = fp32(row)).  drain=True adds advance_beam's
    length-cap drain (bb/search.py:227-229)."""
    if not beam.candidates:
        raise InvariantViolation("cannot expand an empty beam")
    nact = beam.active_width()
    if str(getattr(config.policy, "value", config.policy)) == "immediate" and nact != len(beam.candidates):
        raise InvariantViolation("immediate policy never keeps finalized candidates on the beam")
    if len(score_rows) != nact:
        raise InvariantViolation(f"expected {nact} score rows, got {len(score_rows)}")
    for row in score_rows:
        if len(row) != vocab.size:
            raise InvariantViolation(
                f"score row of length {len(row)} for vocabulary of size {vocab.size}")
    cfg1 = DecodeConfig(k=config.k, n=1, epsilon=config.epsilon, delta=config.delta,
                        max_candidates=config.max_candidates, max_len=config.max_len,
                        policy=config.policy)
    eng = SearchEngine(cfg1, vocab)
    eng.cfg.no_drain = 0 if drain else 1
    eng.load_corpus([[vocab.sos]])
    _load_beam(eng, beam)
    rows = torch.tensor(np.asarray(score_rows, dtype=np.float64).reshape(nact, vocab.size),
                        dtype=torch.float32).to(eng.device)
    if nact:
        eng.row_topm(rows, N.VS_DTYPE_F32 | N.VS_ROWS_NORMALIZED, nact, nact)
    eng.beam_step()
    t = eng.t
    if int(t["counters"][3]):  # device-detected contract break (bb/search.py:155-158 etc.)
        raise InvariantViolation(f"beam step error {int(t['counters'][3])}")
    k, L = eng.k, eng.max_len
    width = int(t["slot_width"][0])
    emitted_total = int(t["slot_emitted"][0])
    sc = t["c_score"][:width].cpu().numpy()
    ln = t["c_len"][:width].cpu().numpy()
    rw = t["c_row"][:width].cpu().numpy()
    fz = t["c_fin"][:width].cpu().numpy()
    hist = t["hist"].view(k, L).cpu().numpy()
    nxt = tuple(Candidate(tuple(int(x) for x in hist[rw[j], : ln[j]]), float(sc[j]), bool(fz[j]),
                          beam.input_id) for j in range(width))
    res = eng.results()
    emitted = [Candidate(c.tokens, c.score, True, beam.input_id)
               for c in res[0][beam.emitted:emitted_total]]
    # results() marks emitted candidates finalized; a length-cap straggler is
    # emitted with finalized=True by the reference too (bb/search.py:194).
    return Beam(beam.input_id, nxt, beam.l_t + 1, emitted_total), emitted
