"""Device-resident VarStream engine: one refilling batch per GPU.

Replaces the body of the reference driver (bb/scheduler.py:243-287 `_drive`
and `_execute_step` :168-205).  All beam state lives in HBM in the SoA layout
of include/varstream.h; the host only launches kernels and reads a small
status record per step:

    vs_schedule   (K3)  stable removal of finished beams, ε-refill, selection,
                        next step's row list                 -> status
    scorer.logits       decoder / synthetic scorer for the R_t rows
    vs_row_lse_topm (K1) fused log-softmax + per-row top-M
    vs_beam_step  (K2)  per-beam merge / δ,M prune / finalise / emit / drain
    scorer.after_step   K4 row-state reorder from K2's copy plan

Two drivers: ``run`` (one status read per step; supports flush, StepEvent
callbacks and traces — the drop-in path) and ``run_async`` (no per-step host
sync: kernels take R_t from device memory and the host trails the device by
a ring of status snapshots; used for throughput).
"""

from __future__ import annotations

import ctypes as C
import itertools
import os
import math
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _native as N
from .core import Candidate, DecodeConfig, FinalizationPolicy, Vocabulary
from .errors import ConfigError, InvariantViolation
from .harness import flatten_checked
from .metrics import CostParams, MetricsReport


@dataclass(frozen=True)
class StepEvent:
    """Observability record per step (bb/scheduler.py:77-88)."""

    timestep: int
    phase: str
    refilled: tuple
    selected: tuple
    expansions: int
    effective_len: int
    finished: tuple
    live_after: tuple


def refill_threshold(config: DecodeConfig) -> int:
    """bb/scheduler.py:237-240: integer form of live <= eps*n."""
    return math.floor(config.epsilon * config.n + 1e-9)


def _candidate(tokens, score, input_id, _new=object.__new__, _set=object.__setattr__, _C=Candidate):
    """Candidate(tokens, score, True, input_id) without the frozen-dataclass
    __init__ (the bulk materialisation of a decode's outputs)."""
    c = _new(_C)
    _set(c, "tokens", tokens)
    _set(c, "score", score)
    _set(c, "finalized", True)
    _set(c, "input_id", input_id)
    return c


class Harvest:
    """Brings a decode's outputs to the host as ``list[list[Candidate]]``
    (bb/scheduler.py:287) WHILE the device is still decoding.

    Emissions append their tokens to the ``out_tok`` buffer (one atomic per
    beam, csrc/beam_step.cu), and every status snapshot carries the append
    fill and MINLIVE, below which every input has finished (arrival order is
    input order and removal is stable).  So whenever the sync-free driver
    consumes a snapshot whose MINLIVE has advanced by ``chunk`` inputs, the
    outputs of those inputs plus the tokens appended since the last request
    are copied to pinned memory on the engine's stream (behind the kernels
    that wrote them), and chunks whose copies have landed are turned into
    Candidate lists — host work that overlaps the device's remaining steps.
    The bytes moved are exactly the emitted outputs."""

    def __init__(self, eng: "SearchEngine", out: list, gids=None, chunk: int = 256):
        self.eng, self.out, self.gids, self.chunk = eng, out, gids, chunk
        self.lo = 0          # inputs [0, lo) requested
        self.tok_hi = 0      # out_tok[0, tok_hi) requested
        self.toks = np.empty(1 << 16, dtype=np.int32)  # host copy of out_tok[0, landed)
        self.landed = 0
        self.gids_np = None if gids is None else np.ascontiguousarray(np.asarray(gids), dtype=np.int64)
        self.mat = N.load_vsmat()
        self.mat.reserve(eng.vocab.size)
        self.pending = []
        self.d2h_bytes = 0

    def offer(self, st) -> None:
        """A status snapshot consumed by the driver (it is at most ring steps old)."""
        hi = int(st[N.ST_MINLIVE])
        if hi - self.lo >= self.chunk:
            self._request(hi, int(st[N.ST_TOKFILL]))
        self.poll()

    def _request(self, hi: int, fill: int, compact: bool = False) -> None:
        t, k, lo = self.eng.t, self.eng.k, self.lo
        if compact:  # only the emitted candidates' metadata (a device sync: used once the run is over)
            cnt = t["out_count"][lo:hi]
            emitted = (torch.arange(k, device=cnt.device)[None, :] < cnt[:, None]).reshape(-1)
            src = (cnt, t["out_len"][lo * k:hi * k][emitted], t["out_score"][lo * k:hi * k][emitted],
                   t["out_off"][lo * k:hi * k][emitted], t["out_tok"][self.tok_hi:fill])
        else:
            src = (t["out_count"][lo:hi], t["out_len"][lo * k:hi * k], t["out_score"][lo * k:hi * k],
                   t["out_off"][lo * k:hi * k], t["out_tok"][self.tok_hi:fill])
        host = tuple(torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in src)
        for h, x in zip(host, src):
            h.copy_(x, non_blocking=True)
            self.d2h_bytes += h.numel() * h.element_size()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.eng.device))
        self.pending.append((ev, lo, hi, host, 0 if compact else k))
        self.lo, self.tok_hi = hi, fill

    def poll(self, block: bool = False) -> None:
        while self.pending and (block or self.pending[0][0].query()):
            ev, lo, hi, host, stride = self.pending.pop(0)
            ev.synchronize()
            count, lens, scores, offs, tok = (h.numpy() for h in host)
            end = self.landed + tok.shape[0]
            if end > self.toks.shape[0]:
                grown = np.empty(max(end, 2 * self.toks.shape[0]), dtype=np.int32)
                grown[: self.landed] = self.toks[: self.landed]
                self.toks = grown
            self.toks[self.landed:end] = tok
            self.landed = end
            # C: Candidate objects with their slots filled directly (hostsrc/vsmat.c)
            self.mat.fill(self.out, self.gids_np, lo, count, lens, scores, offs, self.toks[:end], stride,
                          Candidate)

    def finish(self, st) -> list:
        """After the run's final status (synchronised): request the rest, wait."""
        fill = int(st[N.ST_TOKFILL])
        if self.lo < self.eng.N or fill > self.tok_hi:
            self._request(self.eng.N, fill, compact=True)
        self.poll(block=True)
        return self.out


class SearchEngine:
    """Owns the device state of one refilling batch (n beam slots x k rows)."""

    def __init__(self, config: DecodeConfig, vocab: Vocabulary, *, device=None,
                 m_rows: int | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2010_02164_b200 requires a CUDA device (sm_100a); "
                               "there is no CPU fallback")
        if config.k > N.VS_MAX_K or config.n > N.VS_MAX_SLOTS or config.max_candidates > N.VS_MAX_M:
            raise ConfigError(f"k<= {N.VS_MAX_K}, n <= {N.VS_MAX_SLOTS}, M <= {N.VS_MAX_M} "
                              "in this build")
        self.lib = N.load_library()
        self.config, self.vocab = config, vocab
        self.device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
        k, n, L = config.k, config.n, config.max_len
        self.k, self.n, self.max_len = k, n, L
        self.capacity = min(config.capacity, n * k)  # a step can never need more rows
        # a step plans at most one copy per surviving child: <= k per selected beam
        self.max_copies = n * k
        immediate = config.policy is FinalizationPolicy.IMMEDIATE
        if immediate and 2 * config.k + 2 > N.VS_MAX_M:
            raise ConfigError(f"immediate policy needs 2k+2 <= {N.VS_MAX_M}")
        # immediate ranks each parent's top-(2k+1) by sum, + 1 sentinel (bb/search.py:159-166)
        # + up to 6 slack entries that settle fp64 ties at the boundary (beam_step.cu)
        slack = max(0, min(6, N.VS_MAX_M - (2 * config.k + 2)))
        self.m_rows = m_rows or (min(2 * config.k + 2 + slack, vocab.size) if immediate
                                 else min(config.max_candidates, vocab.size))
        dev = self.device
        i32 = dict(dtype=torch.int32, device=dev)
        z = torch.zeros
        self.t = {
            "slot_input": z(n, **i32), "slot_lt": z(n, **i32), "slot_emitted": z(n, **i32),
            "slot_width": z(n, **i32), "slot_active": z(n, **i32), "slot_src_len": z(n, **i32),
            "slot_flags": z(n, **i32), "slot_seed": z(n, dtype=torch.int64, device=dev),
            "c_score": z(n * k, dtype=torch.float64, device=dev), "c_len": z(n * k, **i32),
            "c_row": z(n * k, **i32), "c_fin": z(n * k, dtype=torch.uint8, device=dev),
            "c_hash": z(n * k, dtype=torch.int64, device=dev), "hist": z(n * k * L, **i32),
            "live": z(n, **i32), "counters": z(8, **i32), "sel": z(n, **i32),
            "sel_off": z(n + 1, **i32), "row_slot": z(self.capacity, **i32),
            "row_cand": z(self.capacity, **i32), "row_phys": z(self.capacity, **i32),
            "row_len": z(self.capacity, **i32),
            "top_tok": z(self.capacity * self.m_rows, **i32),
            "top_logp": z(self.capacity * self.m_rows, dtype=torch.float32, device=dev),
            "row_lse": z(self.capacity, dtype=torch.float32, device=dev),
            "copy_list": z(n * k * 3, **i32), "n_copy": z(1, **i32),
            "status": z(N.status_ints(n), **i32), "fallbacks": z(1, **i32),
            "c_act": z(n * k, **i32),
        }
        self.status_host = torch.zeros(N.status_ints(n), dtype=torch.int32, pin_memory=True)
        self.cfg = N.VsConfig(k=k, n=n, max_candidates=config.max_candidates, max_len=L,
                              vocab_size=vocab.size, sos=vocab.sos, eos=vocab.eos,
                              policy=N.VS_POLICY_IMMEDIATE if immediate else N.VS_POLICY_DEFERRED,
                              capacity=self.capacity,
                              refill_threshold=refill_threshold(config), delta=config.delta)
        self.state = N.VsState()
        for f in N.STATE_FIELDS:
            if f in self.t:
                setattr(self.state, f, self.t[f].data_ptr())
        self.N = 0
        self._k1_ws = None
        self._pinned = {}  # reusable pinned D2H buffers (results)
        self._hdr = None   # pinned status ring of the sync-free driver
        self._bufs = {}    # grow-only corpus / output buffers
        self._forks = {}   # scorer forks bound to this engine (concurrent batches)
        self._graphs, self._graph_key, self._graph_scorer = None, None, None
        self._sp = None    # stream pinned by the running driver

    # ------------------------------------------------------------------ data
    @property
    def stream_ptr(self) -> int:
        # the drivers pin the stream for their launches (one query per step, not per call)
        sp = self._sp
        return sp if sp is not None else torch.cuda.current_stream(self.device).cuda_stream

    def load_corpus(self, corpus, *, src_tok=None, src_off=None) -> None:
        """Copy the (length-bucketed) input stream to HBM and size the outputs.
        Pass ``src_tok``/``src_off`` (pinned host or device int32) to skip the
        Python flattening."""
        if src_off is None:
            src_tok, src_off = flatten_checked(corpus, self.vocab.size)  # bb/model.py:90-102, before any launch
        if isinstance(src_off, np.ndarray):
            src_off, src_tok = torch.from_numpy(src_off), torch.from_numpy(src_tok)
        n_in = int(src_off.shape[0]) - 1
        if n_in < 1:
            raise ConfigError("corpus must be nonempty")
        self.N = n_in
        dev = self.device
        if not src_tok.numel():
            src_tok = torch.zeros(1, dtype=torch.int32)
        # host inputs land in grow-only device buffers, so device pointers (and
        # the captured step graphs that hold them) stay valid across calls
        self.t["src_off"] = src_off if src_off.is_cuda else self._grow("src_off", src_off)
        self.t["src_tok"] = src_tok if src_tok.is_cuda else self._grow("src_tok", src_tok)
        k, L = self.k, self.max_len
        if n_in * k * L >= 2 ** 31:
            raise ConfigError(f"{n_in} inputs x k={k} x max_len={L} exceeds one engine's int32 token "
                              "offsets; shard the corpus (streams / ranks)")
        for f, n, dt in (("out_count", n_in, torch.int32), ("out_len", n_in * k, torch.int32),
                         ("out_score", n_in * k, torch.float64), ("out_off", n_in * k, torch.int32),
                         ("out_tok", n_in * k * L, torch.int32)):
            buf = self._bufs.get(f)
            if buf is None or buf.numel() < n:  # only emitted entries are ever read
                buf = self._bufs[f] = torch.empty(n, dtype=dt, device=dev)
            self.t[f] = buf[:n]
        for f in ("src_off", "src_tok", "out_count", "out_len", "out_score", "out_off", "out_tok"):
            setattr(self.state, f, self.t[f].data_ptr())

    def _grow(self, name: str, src: torch.Tensor) -> torch.Tensor:
        buf = self._bufs.get(name)
        n = src.numel()
        if buf is None or buf.numel() < n:
            buf = self._bufs[name] = torch.empty(n + n // 4, dtype=src.dtype, device=self.device)
        view = buf[:n]
        view.copy_(src, non_blocking=True)
        return view

    def results(self, out: list | None = None, gids=None) -> list:
        """The run's outputs as list[list[Candidate]] in input order
        (bb/scheduler.py:287): one D2H of the emitted outputs (the append
        buffer's fill comes from the final status)."""
        st = self.read_status().copy()
        st[N.ST_TOKFILL] = int(self.t["counters"][6].item())  # authoritative fill (any driver)
        h = Harvest(self, out if out is not None else [[] for _ in range(self.N)], gids, chunk=1 << 30)
        res = h.finish(st)
        self.last_d2h_bytes = h.d2h_bytes
        return res

    def packed(self):
        """Emitted outputs packed in local input order, on the device:
        (count [N] i32, lens [E] i32, scores [E] f64, tokens [T] i32) — what
        the multi-GPU gather ships (parallel.gather_results)."""
        t, k, n_in, dev = self.t, self.k, self.N, self.device
        count = t["out_count"][:n_in]
        emitted = (torch.arange(k, device=dev)[None, :] < count[:, None]).reshape(-1)
        lens = t["out_len"][: n_in * k][emitted]
        scores = t["out_score"][: n_in * k][emitted]
        offs = t["out_off"][: n_in * k][emitted].long()
        total = int(lens.sum().item())
        seg = torch.repeat_interleave(torch.arange(lens.numel(), device=dev), lens.long(), output_size=total)
        starts = torch.cumsum(lens.long(), 0) - lens.long()
        idx = offs[seg] + (torch.arange(total, device=dev) - starts[seg])
        return count.to(torch.int32), lens.to(torch.int32), scores, t["out_tok"][idx].to(torch.int32)

    # --------------------------------------------------------------- kernels
    def schedule(self, *, first: bool, remove: bool, admit: int, select: int, mirror: int | None = None) -> None:
        """Standalone K3 (first schedule of a run, flush transitions)."""
        N.check(self.lib.vs_schedule_mirror(C.byref(self.cfg), C.byref(self.state), self.N, int(first),
                                            int(remove), admit, select, mirror, self.stream_ptr),
                "vs_schedule_mirror")

    def read_status(self) -> np.ndarray:
        self.status_host.copy_(self.t["status"], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        st = self.status_host.numpy()
        if st[N.ST_ERROR] == N.VS_ERR_CONFIG:
            raise ConfigError("a single beam needs more expansions than the step capacity")
        if st[N.ST_ERROR]:
            raise InvariantViolation(f"device scheduler error {int(st[N.ST_ERROR])}")
        return st

    def row_topm(self, logits: torch.Tensor, dtype_code: int, R_host: int, R_grid: int,
                 d_R: int | None = None) -> None:
        ld = logits.stride(0)
        if dtype_code & 0xff == N.VS_DTYPE_F64:
            # reference fp64 log-prob rows: exact values go to the beam step
            if "top_logp64" not in self.t:
                self.t["top_logp64"] = torch.zeros(self.capacity * self.m_rows, dtype=torch.float64,
                                                   device=self.device)
            self.state.top_logp64 = self.t["top_logp64"].data_ptr()
            N.check(self.lib.vs_row_topm_f64(
                logits.data_ptr(), ld, self.vocab.size, self.m_rows, R_host, d_R, R_grid,
                self.t["top_tok"].data_ptr(), self.t["top_logp"].data_ptr(),
                self.t["top_logp64"].data_ptr(), self.stream_ptr), "vs_row_topm_f64")
            return
        self.state.top_logp64 = None
        nbytes = int(self.lib.vs_row_lse_topm_ws_bytes(self.capacity, self.vocab.size, dtype_code))
        ws = self._k1_ws
        if ws is None or ws.numel() < nbytes:  # zeroed once; counters self-reset
            ws = self._k1_ws = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        N.check(self.lib.vs_row_lse_topm_ws(
            logits.data_ptr(), dtype_code, ld, self.vocab.size, self.m_rows, R_host, d_R, R_grid,
            self.t["top_tok"].data_ptr(), self.t["top_logp"].data_ptr(), self.t["row_lse"].data_ptr(),
            self.t["fallbacks"].data_ptr(), ws.data_ptr(), ws.numel(), self.stream_ptr),
            "vs_row_lse_topm_ws")

    def beam_step(self) -> None:
        N.check(self.lib.vs_beam_step(C.byref(self.cfg), C.byref(self.state), self.m_rows,
                                      self.stream_ptr), "vs_beam_step")

    _FUSED = os.environ.get("VS_FUSED_SCHED", "1") != "0"

    def beam_step_schedule(self, *, admit: int, select: int, mirror: int | None = None) -> None:
        """K2 with K3 fused into its last CTA: this step's prune/finalise plus
        the next step's removal, refill, selection and row list (VS_FUSED_SCHED=0:
        the same work as two launches, K2 then the standalone K3)."""
        if self._FUSED:
            N.check(self.lib.vs_beam_step_schedule(C.byref(self.cfg), C.byref(self.state), self.m_rows, self.N,
                                                   admit, select, mirror, self.stream_ptr),
                    "vs_beam_step_schedule")
        else:
            self.beam_step()
            self.schedule(first=False, remove=True, admit=admit, select=select, mirror=mirror)

    def status_ptr(self, idx: int) -> int:
        return self.t["status"].data_ptr() + 4 * idx

    # ---------------------------------------------------------------- drivers
    def _step(self, scorer, st: np.ndarray, *, phase: str, admit: int, select: int) -> None:
        """One timestep: scorer, K1, then K2 with the NEXT step's schedule
        (modes admit/select) fused into its last CTA, then the scorer's K4."""
        R = int(st[N.ST_R])
        if st[N.ST_NADMIT] > 0:
            scorer.on_admit(self, st)
        logits, code = scorer.logits(self, R)
        if code != N.VS_K1_DONE:
            self.row_topm(logits, code, R, R)
        else:
            self.state.top_logp64 = None
        self.beam_step_schedule(admit=admit, select=select)
        scorer.after_step(self, R)

    def run(self, corpus, scorer, *, admit_mode: int, select_mode: int, flush_enabled: bool,
            trace: bool = False, on_step: Callable | None = None):
        """Synchronous driver mirroring bb/scheduler.py:243-287 step for step.
        The schedule that opens iteration t+1 (removal of step t's finished
        beams, flush check, refill, selection) runs inside step t's fused
        beam-step launch, so the host decides its modes before launching."""
        self._sp = None
        cfgd = self.config
        self.load_corpus(corpus)
        scorer.bind(self)
        self._sp = torch.cuda.current_stream(self.device).cuda_stream
        try:
            return self._run(scorer, admit_mode, select_mode, flush_enabled, trace, on_step)
        finally:
            self._sp = None

    def _run(self, scorer, admit_mode, select_mode, flush_enabled, trace, on_step):
        cfgd = self.config
        report = MetricsReport.new(trace=trace)
        cost = CostParams(cfgd.cost_c0, cfgd.cost_c1)
        n = self.n
        timestep = 0
        next_flush = cfgd.flush_interval if flush_enabled and cfgd.flush_interval else None
        pending = None  # event fields of the last executed step, awaiting removal info
        FLUSH = (N.VS_ADMIT_NONE, N.VS_SELECT_ALL)
        STREAM = (admit_mode, select_mode)

        def close_event(st):
            nonlocal pending
            if pending is not None and on_step is not None:
                h = N.ST_HDR
                fin = tuple(int(x) for x in st[h + n:h + n + st[N.ST_NFIN]])
                live = tuple(int(x) for x in st[h + 2 * n:h + 2 * n + st[N.ST_NLIVE_AFTER]])
                on_step(StepEvent(*pending, fin, live))
            pending = None

        def execute(st, phase, refilled, nxt):
            nonlocal timestep, pending
            self._step(scorer, st, phase=phase, admit=nxt[0], select=nxt[1])
            timestep += 1
            R, L = int(st[N.ST_R]), int(st[N.ST_L])
            report.record_step(R, L, cost)
            sel = tuple(int(x) for x in st[N.ST_HDR:N.ST_HDR + st[N.ST_NSEL]])
            pending = (timestep, phase, refilled, sel, R, L)
            st2 = self.read_status()
            close_event(st2)
            return st2

        # the first iteration's top (bb/scheduler.py:261-270); flush_interval >= 1
        phase = "stream"
        self.schedule(first=True, remove=False, admit=admit_mode, select=select_mode)
        st = self.read_status()
        while True:
            if phase == "flush":  # bb/scheduler.py:262-265 flush_all: drain every live beam
                if st[N.ST_NLIVE] > 0:
                    st = execute(st, "flush", (), FLUSH)
                    continue
                next_flush = timestep + cfgd.flush_interval
                phase = "stream"
                self.schedule(first=False, remove=False, admit=admit_mode, select=select_mode)
                st = self.read_status()
            if st[N.ST_NLIVE] == 0:
                break
            a0, na = int(st[N.ST_ADMIT0]), int(st[N.ST_NADMIT])
            flush_next = next_flush is not None and timestep + 1 >= next_flush
            st = execute(st, "stream", tuple(range(a0, a0 + na)), FLUSH if flush_next else STREAM)
            phase = "flush" if flush_next else "stream"
        if st[N.ST_CURSOR] != self.N:
            raise InvariantViolation(f"run consumed {int(st[N.ST_CURSOR])} of {self.N} inputs")
        return self.results(), report

    def async_steps(self, corpus=None, scorer=None, *, admit_mode: int, select_mode: int, ring: int = 16,
                    trace: bool = False, src_tok=None, src_off=None, k1_events: list | None = None,
                    steps_per_graph: int | None = None, harvest_into: list | None = None, gids=None,
                    harvest_chunk: int = 256):
        """Generator form of the host-sync-free driver: every ``next()``
        launches a few steps (on the CUDA stream current at that call) and
        consumes status snapshots ``ring`` steps behind; it returns the
        MetricsReport (StopIteration.value).  Several engines' generators can
        be interleaved on separate streams (``drive_concurrent``).

        Step l runs the scorer, K1 and the fused beam-step kernel, whose last
        CTA schedules step l+1 and writes that status header straight into
        pinned slot hdr[(l+1) % ring] (no copy launch).  With a graph-safe
        scorer, ``steps_per_graph`` consecutive steps are one CUDA graph
        replay (programmatic dependent launch chains every kernel, across
        steps too); the device keeps stepping past the end of the stream
        with empty steps until the host sees the final snapshot.

        With ``harvest_into`` (a list indexed by global input id; ``gids`` maps
        this engine's inputs to global ids) the outputs are streamed to the
        host while the device decodes (``Harvest``)."""
        self._sp = None
        cfgd = self.config
        self.load_corpus(corpus, src_tok=src_tok, src_off=src_off)
        scorer.bind(self)
        report = MetricsReport.new(trace=trace)
        cost = CostParams(cfgd.cost_c0, cfgd.cost_c1)
        graphed = getattr(scorer, "graph_safe", False)
        if steps_per_graph is None:
            steps_per_graph = int(os.environ.get("VS_STEPS_PER_GRAPH", "8"))
        # K1 timing (k1_events): one step per graph, timing events captured around
        # K1 as graph nodes, read back as each step's snapshot is consumed
        spg = max(1, steps_per_graph) if graphed and k1_events is None else 1
        ring = max(ring, 2 * spg)
        ring += (-ring) % spg  # a multiple of spg: graph g always writes the same slots
        if self._hdr is None or self._hdr.shape[0] != ring:
            self._hdr = torch.zeros((ring, N.ST_HDR), dtype=torch.int32, pin_memory=True)
        hdr = self._hdr
        harvest = Harvest(self, harvest_into, gids, harvest_chunk) if harvest_into is not None else None
        events = [torch.cuda.Event() for _ in range(ring)]
        cap = self.capacity
        d_R = self.status_ptr(N.ST_R)
        launched = processed = 0
        graphs = self._step_graphs(scorer, ring, spg, admit_mode, select_mode,
                                   k1_timing=k1_events is not None) if graphed else None
        stream = torch.cuda.current_stream(self.device)
        self.schedule(first=True, remove=False, admit=admit_mode, select=select_mode, mirror=hdr[0].data_ptr())
        events[0].record(stream)
        done = False
        while not done:
            # launching steps launched..launched+spg-1 overwrites snapshot slots
            # up to launched+spg: everything older than that must be consumed
            while launched + spg - processed >= ring:
                events[processed % ring].synchronize()
                if graphs is not None and k1_events is not None and processed >= 1:
                    e0, e1 = self._graph_events[(processed - 1) % len(graphs)]
                    k1_events.append(e0.elapsed_time(e1))  # step processed-1 has completed
                st = hdr[processed % ring].numpy()
                if st[N.ST_ERROR]:
                    self.read_status()
                if st[N.ST_NLIVE] == 0:
                    done = True
                    break
                report.record_step(int(st[N.ST_R]), int(st[N.ST_L]), cost)
                processed += 1
                if harvest is not None:
                    harvest.offer(st)
            if done:
                break
            stream = torch.cuda.current_stream(self.device)
            self._sp = stream.cuda_stream
            if graphs is not None:
                graphs[(launched // spg) % len(graphs)].replay()
            else:
                scorer.on_admit(self, None)
                logits, code = scorer.logits(self, None)
                if k1_events is not None:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                if code != N.VS_K1_DONE:
                    self.row_topm(logits, code, 0, cap, d_R)
                if k1_events is not None:
                    e1.record(stream)
                    e1.synchronize()
                    k1_events.append(e0.elapsed_time(e1))
                self.beam_step_schedule(admit=admit_mode, select=select_mode,
                                        mirror=hdr[(launched + 1) % ring].data_ptr())
                scorer.after_step(self, None)
            for q in range(1, spg + 1):
                events[(launched + q) % ring].record(stream)
            launched += spg
            yield
        self.launched_steps = launched
        self._sp = None
        st = self.read_status()
        if st[N.ST_CURSOR] != self.N:
            raise InvariantViolation(f"run consumed {int(st[N.ST_CURSOR])} of {self.N} inputs")
        if harvest is not None:
            harvest.finish(st)
            self.last_d2h_bytes = harvest.d2h_bytes
        return report

    def _step_graphs(self, scorer, ring: int, spg: int, admit_mode: int, select_mode: int,
                     k1_timing: bool = False):
        """Capture (once per engine state / scorer binding) ring/spg graphs of
        spg steps each: scorer launches, K1, K2+K3 (status header -> the next
        pinned slot).  k1_timing: external timing events around each K1 as
        graph nodes (spg = 1), so K1 is timed on the device with no host gaps."""
        # the graphs bake in the scorer's parameters and buffer addresses: key on
        # the scorer object itself (held strongly, compared with `is`, so a
        # recycled id() can never match) plus its graph_key() (parameters and
        # data pointers, which change when bind() reallocates)
        gk = scorer.graph_key() if hasattr(scorer, "graph_key") else None
        key = (gk, ring, spg, admit_mode, select_mode, k1_timing, self.N,  # N is a K3 launch argument
               tuple(getattr(self.state, f) for f in N.STATE_FIELDS), self._hdr.data_ptr())
        if self._graph_key == key and self._graph_scorer is scorer:
            return self._graphs
        cap, d_R = self.capacity, self.status_ptr(N.ST_R)
        nbytes = int(self.lib.vs_row_lse_topm_ws_bytes(cap, self.vocab.size, N.VS_DTYPE_F32))
        if self._k1_ws is None or self._k1_ws.numel() < nbytes:  # allocate outside the capture
            self._k1_ws = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        torch.cuda.current_stream(self.device).synchronize()
        graphs, gev = [], []
        for gi in range(ring // spg):
            g = torch.cuda.CUDAGraph()
            if k1_timing:
                gev.append((torch.cuda.Event(enable_timing=True, external=True),
                            torch.cuda.Event(enable_timing=True, external=True)))
            with torch.cuda.graph(g):
                for q in range(spg):
                    step = gi * spg + q
                    scorer.on_admit(self, None)
                    logits, code = scorer.logits(self, None)
                    if k1_timing:
                        gev[-1][0].record()
                    if code != N.VS_K1_DONE:
                        self.row_topm(logits, code, 0, cap, d_R)
                    if k1_timing:
                        gev[-1][1].record()
                    self.beam_step_schedule(admit=admit_mode, select=select_mode,
                                            mirror=self._hdr[(step + 1) % ring].data_ptr())
                    scorer.after_step(self, None)
            graphs.append(g)
        self._graphs, self._graph_key, self._graph_scorer = graphs, key, scorer
        self._graph_events = gev
        return graphs

    def run_async(self, corpus=None, scorer=None, *, admit_mode: int, select_mode: int,
                  ring: int = 16, trace: bool = False, src_tok=None, src_off=None,
                  materialize: bool = True, k1_events: list | None = None):
        """Host-sync-free driver (no flush / no StepEvents): every kernel reads
        R_t from device memory, status headers are streamed into a pinned ring
        and consumed `ring` steps behind the device."""
        n_in = len(corpus) if corpus is not None else int(src_off.shape[0]) - 1
        out = [[] for _ in range(n_in)] if materialize else None
        gen = self.async_steps(corpus, scorer, admit_mode=admit_mode, select_mode=select_mode, ring=ring,
                               trace=trace, src_tok=src_tok, src_off=src_off, k1_events=k1_events,
                               harvest_into=out)
        while True:
            try:
                next(gen)
            except StopIteration as stop:
                report = stop.value
                break
        return out, report


def drive_concurrent(jobs):
    """Interleave several engines' sync-free drivers, each on its own CUDA
    stream, one step per engine per round: independent refilling batches share
    the GPU, so one batch's latency-bound kernels (beam step, scheduler, small
    steps) overlap another's streaming ones.  ``jobs`` = [(stream, generator)];
    returns the MetricsReports in job order."""
    reports = [None] * len(jobs)
    live = list(range(len(jobs)))
    while live:
        for j in list(live):
            stream, gen = jobs[j]
            with torch.cuda.stream(stream):
                try:
                    next(gen)
                except StopIteration as stop:
                    reports[j] = stop.value
                    live.remove(j)
    return reports
