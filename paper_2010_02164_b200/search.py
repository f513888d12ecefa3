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


_EXPAND_ENGINES: dict = {}


def _expand_engine(config: DecodeConfig, vocab: Vocabulary, n_beams: int, drain: bool) -> SearchEngine:
    """A cached engine with >= n_beams slots for per-beam expansion calls."""
    n = 1 << max(0, (n_beams - 1).bit_length())
    key = (config.k, config.max_candidates, config.delta, config.max_len, str(config.policy),
           vocab.size, vocab.sos, vocab.eos, n, torch.cuda.current_device())
    eng = _EXPAND_ENGINES.pop(key, None)
    if eng is None:
        while len(_EXPAND_ENGINES) >= 16:  # a small LRU: per-beam callers reuse a few shapes
            _EXPAND_ENGINES.pop(next(iter(_EXPAND_ENGINES)))
        cfg = DecodeConfig(k=config.k, n=n, epsilon=config.epsilon, delta=config.delta,
                           max_candidates=config.max_candidates, max_len=config.max_len, policy=config.policy)
        eng = SearchEngine(cfg, vocab)
    _EXPAND_ENGINES[key] = eng
    eng.cfg.no_drain = 0 if drain else 1
    return eng


def _load_beams(eng: SearchEngine, beams) -> list[int]:
    """Write beam b into slot b (slot_input = b, its emissions go to output
    row b); returns the active widths.  One H2D per field."""
    k, L, B = eng.k, eng.max_len, len(beams)
    eng.load_corpus([[0]] * B)
    widths = [len(b.candidates) for b in beams]
    nact = [b.active_width() for b in beams]
    hist = np.zeros((B, k, L), dtype=np.int32)
    score = np.zeros((B, k), dtype=np.float64)
    clen = np.zeros((B, k), dtype=np.int32)
    fin = np.zeros((B, k), dtype=np.uint8)
    for b, beam in enumerate(beams):
        for j, c in enumerate(beam.candidates):
            hist[b, j, : len(c.tokens)] = c.tokens
            score[b, j], clen[b, j], fin[b, j] = c.score, len(c.tokens), int(c.finalized)
    t, dev = eng.t, eng.device
    i32 = lambda x: torch.tensor(x, dtype=torch.int32)  # noqa: E731
    t["slot_input"][:B] = i32(list(range(B))).to(dev)
    t["slot_lt"][:B] = i32([b.l_t for b in beams]).to(dev)
    t["slot_emitted"][:B] = i32([b.emitted for b in beams]).to(dev)
    t["slot_width"][:B] = i32(widths).to(dev)
    t["slot_active"][:B] = i32(nact).to(dev)
    t["slot_flags"][:B] = 1
    t["hist"].view(-1, k, L)[:B].copy_(torch.from_numpy(hist))
    t["c_score"].view(-1, k)[:B].copy_(torch.from_numpy(score))
    t["c_len"].view(-1, k)[:B].copy_(torch.from_numpy(clen))
    t["c_row"].view(-1, k)[:B] = torch.arange(k, dtype=torch.int32, device=dev)
    t["c_fin"].view(-1, k)[:B].copy_(torch.from_numpy(fin))
    st = np.zeros(N.status_ints(eng.n), dtype=np.int32)
    st[N.ST_R], st[N.ST_NSEL] = sum(nact), B
    t["status"].copy_(torch.from_numpy(st))
    t["sel"][:B] = i32(list(range(B))).to(dev)
    t["sel_off"][: B + 1] = i32(np.concatenate([[0], np.cumsum(nact)]).tolist()).to(dev)
    t["n_copy"].zero_()
    t["counters"].zero_()
    t["out_len"].zero_()  # emission slots below beam.emitted are never written
    t["out_off"].zero_()
    return nact


def expand_beams(beams, score_rows, config: DecodeConfig, vocab: Vocabulary, *, drain: bool = False):
    """bb/search.py:76-103 (expand_beam) for several beams in ONE device step:
    K1-f64 over all their rows, then one beam-step launch (one CTA per beam).
    ``score_rows[b]`` are beam b's per-active-candidate log-prob rows in beam
    order, kept in fp64 end to end (top-M by exact row value, fp64 score
    adds), so each result is the reference's bit for bit.  drain=True adds
    advance_beam's length-cap drain (bb/search.py:227-229).  Returns
    [(next beam, emitted candidates)] in input order."""
    policy_imm = str(getattr(config.policy, "value", config.policy)) == "immediate"
    for beam, rows in zip(beams, score_rows):
        if not beam.candidates:
            raise InvariantViolation("cannot expand an empty beam")
        nact = beam.active_width()
        if policy_imm and nact != len(beam.candidates):
            raise InvariantViolation("immediate policy never keeps finalized candidates on the beam")
        if len(rows) != nact:
            raise InvariantViolation(f"expected {nact} score rows, got {len(rows)}")
        for row in rows:
            if len(row) != vocab.size:
                raise InvariantViolation(
                    f"score row of length {len(row)} for vocabulary of size {vocab.size}")
    if not beams:
        return []
    if len(beams) > N.VS_MAX_SLOTS:
        return [r for b0 in range(0, len(beams), N.VS_MAX_SLOTS)
                for r in expand_beams(beams[b0:b0 + N.VS_MAX_SLOTS], score_rows[b0:b0 + N.VS_MAX_SLOTS],
                                      config, vocab, drain=drain)]
    eng = _expand_engine(config, vocab, len(beams), drain)
    nact = _load_beams(eng, beams)
    R = sum(nact)
    if R:  # the rows' own fp64 values (bb/search.py:69-71): vs_row_topm_f64
        flat = np.asarray([r for rows in score_rows for r in rows], dtype=np.float64).reshape(R, vocab.size)
        eng.row_topm(torch.from_numpy(flat).to(eng.device), N.VS_DTYPE_F64 | N.VS_ROWS_NORMALIZED, R, R)
    eng.beam_step()
    t = eng.t
    if int(t["counters"][3]):  # device-detected contract break (bb/search.py:155-158 etc.)
        raise InvariantViolation(f"beam step error {int(t['counters'][3])}")
    k, L, B = eng.k, eng.max_len, len(beams)
    width = t["slot_width"][:B].cpu().tolist()
    emitted_total = t["slot_emitted"][:B].cpu().tolist()
    sc = t["c_score"].view(-1, k)[:B].cpu().numpy()
    ln = t["c_len"].view(-1, k)[:B].cpu().numpy()
    rw = t["c_row"].view(-1, k)[:B].cpu().numpy()
    fz = t["c_fin"].view(-1, k)[:B].cpu().numpy()
    hist = t["hist"].view(-1, k, L)[:B].cpu().numpy()
    res = eng.results()
    out = []
    for b, beam in enumerate(beams):
        nxt = tuple(Candidate(tuple(int(x) for x in hist[b, rw[b, j], : ln[b, j]]), float(sc[b, j]),
                              bool(fz[b, j]), beam.input_id) for j in range(width[b]))
        # emitted candidates are finalized; a length-cap straggler is emitted
        # with finalized=True by the reference too (bb/search.py:194)
        emitted = [Candidate(c.tokens, c.score, True, beam.input_id)
                   for c in res[b][beam.emitted:emitted_total[b]]]
        out.append((Beam(beam.input_id, nxt, beam.l_t + 1, emitted_total[b]), emitted))
    return out


def expand_beam(beam: Beam, score_rows, config: DecodeConfig, vocab: Vocabulary,
                *, drain: bool = False):
    """Device expand_beam (bb/search.py:76-103): ``expand_beams`` for one beam.
    Returns (next beam, emitted list)."""
    return expand_beams([beam], [score_rows], config, vocab, drain=drain)[0]
