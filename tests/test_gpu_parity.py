"""GPU parity: the sm_100a kernels vs the CPU oracle (pinned to the reference).

All calls go through the C-ABI library (paper_2010_02164_b200/_lib/libvarstream.so).
Contract (BASELINE.json north_star): given identical logits, top-k indices,
prune/finalise decisions and refill order are bit-exact; fp64 scores are
bit-exact given the kernel's exported lse (logp = fp32(logit - lse)); lse
itself agrees with an fp64 log-softmax within 1e-5 relative.
"""
import math

import numpy as np
import pytest

from goldens import fl, load
from oracle import varstream_oracle as O
from oracle.scorers import HashLogitsCPU, LseReplayScorer, SeededHashScorerCPU

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _pkg():
    import paper_2010_02164_b200 as P
    from paper_2010_02164_b200 import _native as N
    from paper_2010_02164_b200.engine import SearchEngine
    from paper_2010_02164_b200.scorers import DeviceHashScorer, HostScorerAdapter, LseRecorder

    return P, N, SearchEngine, DeviceHashScorer, HostScorerAdapter, LseRecorder


def _check_rows(x32: np.ndarray, M: int, tok, lp, lse, normalized=False):
    R, V = x32.shape
    x64 = x32.astype(np.float64)
    for r in range(R):
        l = np.float32(0.0) if normalized else np.float32(lse[r])
        logp = (x32[r] - l).astype(np.float32)
        want = O.row_top_m(logp.astype(np.float64), M)
        m = min(M, V)
        assert list(tok[r, :m]) == list(want), f"row {r}"
        assert np.array_equal(lp[r, :m], logp[want]), f"row {r}"
        if not normalized and np.isfinite(x64[r]).any():
            peak = x64[r].max()
            ref = peak + math.log(np.exp(x64[r] - peak).sum())
            assert abs(float(lse[r]) - ref) <= 1e-5 * max(1.0, abs(ref)), f"row {r} lse"


CASES = [(1000, 3), (1000, 5), (2048, 10), (42024, 5), (42024, 50), (17, 3), (3, 5), (4096, 1),
         (33, 16), (1001, 64), (65535, 5), (65536, 7),  # 32-bit / 64-bit top-list keys
         (4096, 32), (4096, 33)]  # largest register top-list / smallest buffered-candidate M


@pytest.mark.parametrize("kernel", ["split", "warp"])
@pytest.mark.parametrize("V,M", CASES)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_row_topm_matches_oracle(V, M, dtype, kernel):
    P, *_ = _pkg()
    rng = np.random.default_rng(V * 131 + M)
    R = 24
    x = rng.normal(0, 3, (R, V)).astype(np.float32)
    x[1] = np.round(x[1] * 2) / 2             # heavy ties
    x[2] = 0.25                               # uniform row -> exact fallback
    x[3, ::3] = -np.inf                       # masked tokens
    x[4] = x[4] * 1e-3 + 40.0                 # near-equal logits that merge after - lse
    x[5, :] = -np.inf
    x[5, V // 2] = 1.0                        # one finite entry
    x[6] = np.float32(1e6) + x[6]             # large offset
    t = torch.from_numpy(x).cuda()
    if dtype == "bf16":
        t = t.to(torch.bfloat16)
        x = t.float().cpu().numpy()
    tok, lp, lse, fb = P.row_lse_topm(t, M, kernel=kernel)
    torch.cuda.synchronize()
    _check_rows(x, M, tok.cpu().numpy(), lp.cpu().numpy(), lse.cpu().numpy())


def _rows(rng, R, V, kind):
    if kind == "normal":
        return rng.normal(0, 3, (R, V)).astype(np.float32)
    u = rng.random((R, V)).clip(2.0 ** -24)                 # log-like (the decode's scorer)
    return (-0.5 * np.log2(u)).astype(np.float32)


@pytest.mark.parametrize("M", [5, 32])
@pytest.mark.parametrize("R", [1, 3, 37, 600, 2000])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_row_topm_tma_split_rows(R, dtype, M):
    """The TMA split-row kernel at step sizes from 1 row (a row spread over
    many warps) to 2000 rows (whole rows per warp), checked row by row on a
    sample against the oracle (given the kernel's lse)."""
    P, *_ = _pkg()
    rng = np.random.default_rng(R)
    V = 42024
    x = _rows(rng, R, V, "loglike" if R % 2 else "normal")
    t = torch.from_numpy(x).cuda()
    if dtype == "bf16":
        t = t.to(torch.bfloat16)
        x = t.float().cpu().numpy()
    tok, lp, lse, fb = P.row_lse_topm(t, M, kernel="split")
    torch.cuda.synchronize()
    pick = sorted(set(np.linspace(0, R - 1, min(R, 24)).astype(int).tolist()))
    _check_rows(x[pick], M, tok.cpu().numpy()[pick], lp.cpu().numpy()[pick], lse.cpu().numpy()[pick])


@pytest.mark.parametrize("kernel", ["split", "warp"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_row_topm_lse_is_partition_invariant(dtype, kernel):
    """lse (hence every logp) of a row is a function of the row alone: the same
    row scored alone, among 5 rows, among 900 or among 6,400 rows (different
    splits of its segments over warps: the warp kernel picks 8, 4, 2 or 1 warps
    per row from the live row count) gives bit-identical outputs — so an
    input's decode does not depend on what else shares its batch."""
    P, *_ = _pkg()
    V, M = 42024, 5
    g = torch.Generator(device="cuda").manual_seed(11)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    big = (torch.randn((6400, V), generator=g, device="cuda") * 2.0).to(tdt)
    big[450, 7] = 40.0  # a late max raise inside one segment
    outs = []
    for lo, hi in [(450, 451), (448, 453), (0, 900), (300, 1000), (0, 6400)]:
        tok, lp, lse, _ = P.row_lse_topm(big[lo:hi], M, kernel=kernel)
        outs.append((tok[450 - lo].cpu(), lp[450 - lo].cpu(), lse[450 - lo].cpu()))
    for o in outs[1:]:
        assert torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1]) and torch.equal(o[2], outs[0][2])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_row_topm_tma_scalar_tail_and_ties(dtype):
    """Rows whose byte length is not a multiple of 16 (scalar tail on the TMA
    path), ties straddling segment boundaries, and a winner in the tail."""
    P, *_ = _pkg()
    rng = np.random.default_rng(5)
    V, M = 42027, 6
    big = torch.from_numpy(rng.normal(0, 1, (40, 42032)).astype(np.float32)).cuda()
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    big = big.to(tdt)
    view = big[:, :V]
    view[1, V - 1] = 30.0          # winner in the scalar tail
    view[2, 2047:2049] = 9.0       # tie across the first segment boundary (bf16: 2048 elems/seg)
    view[2, 1023:1025] = 9.0       # (f32: 1024 elems/seg)
    view[3, :] = 0.5               # all tied -> exact fallback
    x = view.float().cpu().numpy()
    tok, lp, lse, fb = P.row_lse_topm(view, M, kernel="split")
    torch.cuda.synchronize()
    _check_rows(x, M, tok.cpu().numpy(), lp.cpu().numpy(), lse.cpu().numpy())


def test_row_topm_strided_and_normalized_rows():
    P, *_ = _pkg()
    rng = np.random.default_rng(3)
    big = torch.from_numpy(rng.uniform(-9, 0, (16, 1040)).astype(np.float32)).cuda()
    view = big[:, :1000]  # ld = 1040
    tok, lp, lse, _ = P.row_lse_topm(view, 7, normalized=True)
    _check_rows(view.cpu().numpy(), 7, tok.cpu().numpy(), lp.cpu().numpy(), lse.cpu().numpy(),
                normalized=True)
    assert float(lse.abs().max()) == 0.0


EXPAND = load("expand_cases.json")


def _ocfg(d):
    return O.OConfig(k=d["k"], n=d["n"], epsilon=d["epsilon"], delta=fl(d["delta"]),
                     max_candidates=d["max_candidates"], max_len=d["max_len"], policy=d["policy"])


def _golden_beam(P, case):
    cands = tuple(P.Candidate(tuple(c["tokens"]), fl(c["score"]), c["finalized"])
                  for c in case["beam"]["candidates"])
    return P.Beam(0, cands, case["beam"]["l_t"], case["beam"]["emitted"])


def _check_golden_expand(case, got, emitted, ci):
    w = case["want"]
    key = lambda c: (tuple(c.tokens), c.score, bool(c.finalized))  # noqa: E731
    assert [key(c) for c in got.candidates] == [
        (tuple(c["tokens"]), fl(c["score"]), c["finalized"]) for c in w["next"]], ci
    assert [(c.tokens, c.score) for c in emitted] == [(tuple(c["tokens"]), fl(c["score"])) for c in w["emitted"]], ci
    assert got.emitted == w["emitted_total"] and got.l_t == w["l_t"], ci


def test_device_expand_beam_matches_reference_goldens():
    """Every golden case of the REFERENCE's expand_beam (deferred, incl. the
    row-value pre-truncation gap case, and immediate) through K1-f64 + K2:
    next beam, emissions and every fp64 score bit-identical to the reference's
    own recorded outputs (the rows stay fp64)."""
    P, *_ = _pkg()
    for ci, case in enumerate(EXPAND):
        d, v = case["config"], case["vocab"]
        cfg = P.DecodeConfig(k=d["k"], n=1, delta=fl(d["delta"]), max_candidates=d["max_candidates"],
                             max_len=d["max_len"], policy=d["policy"])
        vocab = P.Vocabulary(v["size"], v["sos"], v["eos"])
        rows = [[fl(x) for x in r] for r in case["rows"]]
        got, emitted = P.expand_beam(_golden_beam(P, case), rows, cfg, vocab)
        _check_golden_expand(case, got, emitted, ci)


def test_expand_beams_batches_many_beams_in_one_step():
    """expand_beams: the golden cases that share a configuration, expanded
    together (one K1-f64 + one beam-step launch), each equal to the reference."""
    import json

    P, *_ = _pkg()
    groups = {}
    for ci, case in enumerate(EXPAND):
        groups.setdefault(json.dumps([case["config"], case["vocab"]], sort_keys=True), []).append(ci)
    big = sorted(groups.values(), key=len)[-6:]
    assert max(len(g) for g in big) >= 3
    for g in big:
        case0 = EXPAND[g[0]]
        d, v = case0["config"], case0["vocab"]
        cfg = P.DecodeConfig(k=d["k"], n=1, delta=fl(d["delta"]), max_candidates=d["max_candidates"],
                             max_len=d["max_len"], policy=d["policy"])
        vocab = P.Vocabulary(v["size"], v["sos"], v["eos"])
        beams = [_golden_beam(P, EXPAND[ci]) for ci in g]
        rows = [[[fl(x) for x in r] for r in EXPAND[ci]["rows"]] for ci in g]
        for ci, (got, emitted) in zip(g, P.expand_beams(beams, rows, cfg, vocab)):
            _check_golden_expand(EXPAND[ci], got, emitted, ci)


def _events(evs):
    return [(e.timestep, e.phase, tuple(e.refilled), tuple(e.selected), e.expansions,
             e.effective_len, tuple(e.finished), tuple(e.live_after)) for e in evs]


class _RefVocabScorer:
    """SeededHashScorerCPU exposing a reference-style .vocab for the adapter."""

    def __init__(self, inner, vocab):
        self.inner, self.vocab = inner, vocab

    def encode(self, tokens, input_id=0):
        return self.inner.encode(tokens, input_id)

    def score_next(self, enc, cand):
        return self.inner.score_next(enc, cand)


RUNS = {f["name"]: f for f in load("runs.json")}


def _golden_events(evs):
    return [(e["timestep"], e["phase"], tuple(e["refilled"]), tuple(e["selected"]), e["expansions"],
             e["effective_len"], tuple(e["finished"]), tuple(e["live_after"])) for e in evs]


@pytest.mark.parametrize("name", sorted(RUNS))
def test_engine_with_reference_scorer_matches_reference_runs(name):
    """The unmodified reference workloads (SeededHashScorer, fp64 log-prob rows)
    driven through the device engine via the drop-in adapter reproduce the
    REFERENCE's own recorded run (tests/golden/runs.json, written by
    oracle/gen_golden.py from bb/scheduler.py): every StepEvent, the per-step
    trace, the simulated cost, and every output token and fp64 score
    bit-exactly (the rows stay fp64 end to end: vs_row_topm_f64)."""
    P, N, SearchEngine, _, HostScorerAdapter, _ = _pkg()
    fx = RUNS[name]
    s = fx["scorer"]
    base = SeededHashScorerCPU(s["vocab_size"], s["sos"], s["eos"], s["seed"], s["eos_bias"])
    d = fx["config"]
    cfg = P.DecodeConfig(k=d["k"], n=d["n"], epsilon=d["epsilon"], delta=fl(d["delta"]),
                         max_candidates=d["max_candidates"], max_len=d["max_len"],
                         capacity=d["capacity"], flush_interval=d["flush_interval"],
                         policy=d["policy"])
    corpus = [tuple(x) for x in fx["corpus"]]
    vocab = P.Vocabulary(s["vocab_size"], s["sos"], s["eos"])
    runner = {"run_varstream": P.run_varstream, "run_varbeam": P.run_varbeam,
              "run_varfifo": P.run_varfifo}[fx["runner"]]
    ev = []
    out, rep = runner(corpus, _RefVocabScorer(base, vocab), cfg, trace=True, on_step=ev.append)
    assert _events(ev) == _golden_events(fx["events"])
    want = [[(tuple(c["tokens"]), fl(c["score"])) for c in per] for per in fx["outputs"]]
    assert [[(c.tokens, c.score) for c in per] for per in out] == want
    r = fx["report"]
    assert rep.timesteps == r["timesteps"] and rep.candidate_expansions == r["candidate_expansions"]
    assert [list(x) for x in rep.per_step_trace] == [list(x) for x in r["trace"]]
    assert rep.simulated_cost == r["simulated_cost"]


def test_row_topm_f64_matches_oracle():
    """K1-f64 (vs_row_topm_f64): top-M of fp64 rows by (value desc, token asc),
    exact values, ties, -inf, NaN never ranked, V < M padding."""
    P, N, *_ = _pkg()
    lib = N.load_library()
    rng = np.random.default_rng(5)
    for R, V, M in ((1, 1, 3), (7, 50, 5), (33, 1000, 12), (5, 4096, 64), (3, 300, 128)):
        x = rng.standard_normal((R, V))
        x[:, ::7] = np.round(x[:, ::7], 1)  # ties
        if V > 4:
            x[0, 1] = -np.inf
            x[-1, 2] = np.nan
        dx = torch.from_numpy(x).cuda()
        tok = torch.empty(R * M, dtype=torch.int32, device="cuda")
        lp = torch.empty(R * M, dtype=torch.float32, device="cuda")
        lp64 = torch.empty(R * M, dtype=torch.float64, device="cuda")
        rc = lib.vs_row_topm_f64(dx.data_ptr(), V, V, M, R, None, R, tok.data_ptr(), lp.data_ptr(),
                                 lp64.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        tok, lp64 = tok.view(R, M).cpu().numpy(), lp64.view(R, M).cpu().numpy()
        for r in range(R):
            order = sorted((t for t in range(V) if x[r, t] == x[r, t]), key=lambda t: (-x[r, t], t))[:M]
            assert list(tok[r, :len(order)]) == order
            assert np.array_equal(lp64[r, :len(order)], x[r, order])
            assert all(tok[r, len(order):] == -1)


def test_greedy_engine_matches_reference_greedy_decode():
    """dispatch_engine("greedy") (batched width-1 beams on the device) gives
    the candidates of bb/search.py:38-49 greedy_decode for every input, and
    the metrics of the reference's unbatched accounting (bb/harness.py:222-238)."""
    P, *_ = _pkg()
    fx = RUNS["c1_varstream_eps0.1667"]
    s = fx["scorer"]
    base = SeededHashScorerCPU(s["vocab_size"], s["sos"], s["eos"], s["seed"], s["eos_bias"])
    d = fx["config"]
    cfg = P.DecodeConfig(k=d["k"], n=d["n"], max_len=d["max_len"])
    corpus = [tuple(x) for x in fx["corpus"]][:80]
    vocab = P.Vocabulary(s["vocab_size"], s["sos"], s["eos"])
    out, rep = P.dispatch_engine("greedy", corpus, _RefVocabScorer(base, vocab), cfg, trace=True)
    ref = base
    want = [O.greedy_decode(ref.encode(x, i), ref, cfg.max_len) for i, x in enumerate(corpus)]
    assert [[(c.tokens, c.score) for c in per] for per in out] == [[(c.tokens, c.score)] for c in want]
    steps = sum(len(c.tokens) - 1 for c in want)
    assert rep.timesteps == steps and rep.candidate_expansions == steps
    assert [(r[1], r[2]) for r in rep.per_step_trace] == [(1, L) for c in want for L in range(1, len(c.tokens))]


HASH_CASES = [
    # name, V, k, n, M, delta, max_len, eps, N, dtype, scale, power, eos_bias[, policy]
    ("toy_c1", 1000, 5, 32, 3, 1.5, 48, 1 / 6, 160, "bf16", 8.0, 1, 6.0),
    ("toy_fixed", 1000, 5, 32, 5, math.inf, 48, 1 / 6, 96, "f32", 8.0, 1, 6.0),
    ("parse_c3", 2048, 10, 64, 3, 10.0, 40, 1 / 6, 120, "bf16", 6.0, 2, 5.0),
    ("wide_k", 3000, 24, 8, 6, 2.0, 20, 1 / 4, 24, "f32", 10.0, 4, 9.0),
    ("wmt_like", 42024, 50, 16, 5, 1.5, 40, 1 / 6, 24, "bf16", 0.5, 0, 7.5),
    ("immediate", 1000, 5, 16, 5, 1.5, 32, 1 / 6, 96, "bf16", 0.5, 0, 4.0, "immediate"),
    ("immediate_k16", 2048, 16, 8, 16, 3.0, 24, 1 / 4, 40, "f32", 0.5, 0, 4.0, "immediate"),
    # edge shapes: one slot x width one; the length cap draining every beam;
    # the build's maximum beam width; many slots with a refill threshold of 0
    ("k1_n1", 1000, 1, 1, 1, math.inf, 12, 1 / 6, 16, "f32", 8.0, 1, 6.0),
    ("len_cap", 1000, 8, 16, 4, 2.0, 3, 1 / 6, 48, "bf16", 0.5, 0, 0.1),
    ("max_k", 600, 128, 4, 8, 4.0, 10, 1 / 6, 12, "f32", 0.5, 0, 3.0),
    ("many_slots", 700, 4, 512, 3, 1.5, 16, 1 / 1024, 700, "bf16", 0.5, 0, 4.0),
]


@pytest.mark.parametrize("case", HASH_CASES, ids=[c[0] for c in HASH_CASES])
def test_device_hash_decode_matches_oracle(case):
    """Whole VarStream decodes with the device scorer: every decision, event and
    fp64 score bit-exact vs the oracle replaying the kernel's lse; the async
    (sync-free) driver reproduces the synchronous one."""
    name, V, k, n, M, delta, ml, eps, Nin, dt, scale, power, eb = case[:13]
    policy = case[13] if len(case) > 13 else "deferred"
    P, N, SearchEngine, DeviceHashScorer, _, LseRecorder = _pkg()
    vocab = P.Vocabulary(V, 0, 2)
    cfg = P.DecodeConfig(k=k, n=n, epsilon=eps, delta=delta, max_candidates=M, max_len=ml,
                         policy=policy)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(99, Nin, V, mean_len=8.0))
    rec = LseRecorder(DeviceHashScorer(vocab, 5, scale=scale, power=power, eos_bias=eb, dtype=dt))
    ev = []
    out, rep = P.run_varstream(corpus, rec, cfg, trace=True, on_step=ev.append)
    cpu = LseReplayScorer(HashLogitsCPU(V, 0, 2, 5, scale=scale, power=power, eos_bias=eb,
                                        dtype=dt), rec.table)
    oev = []
    want, wrep = O.run_varstream(corpus, cpu, O.as_oconfig(cfg), trace=True, on_step=oev.append)
    assert _events(ev) == _events(oev)
    assert [[(c.tokens, c.score) for c in per] for per in out] == O.signature(want)
    assert rep.candidate_expansions == wrep.candidate_expansions
    # sync-free driver: identical outputs and counters
    fast_out, fast_rep = P.run_varstream(
        corpus, DeviceHashScorer(vocab, 5, scale=scale, power=power, eos_bias=eb, dtype=dt), cfg,
        trace=True)
    assert [[(c.tokens, c.score) for c in per] for per in fast_out] == O.signature(want)
    assert fast_rep.per_step_trace == rep.per_step_trace


HASH_LOGIT_CASES = [
    # V, k, n, dtype, scale, power, eos_bias, N: enough rows per step that a
    # CTA walks several rows (grid = column chunks x row groups); tiny V (one
    # chunk, ragged tail group), the WMT vocabulary, every power mode
    (42024, 16, 64, "bf16", 0.5, 0, 7.5, 80),
    (42024, 8, 32, "f32", 0.5, 0, 7.5, 40),
    (1003, 12, 48, "bf16", 8.0, 1, 6.0, 120),
    (5000, 6, 40, "f32", 6.0, 2, 5.0, 80),
    (3001, 6, 40, "bf16", 10.0, 4, 9.0, 80),
]


@pytest.mark.parametrize("case", HASH_LOGIT_CASES, ids=lambda c: f"V{c[0]}_{c[3]}_p{c[5]}")
def test_device_hash_logits_bit_exact(case):
    """Every logit of every scored row (not only the ones that reach a
    decision) equals the CPU mirror oracle/scorers.py:HashLogitsCPU bit for
    bit: admitted rows (inline encode) and extended rows, the EOS column, the
    ragged vocabulary tail."""
    V, k, n, dt, scale, power, eb, Nin = case
    P, N, SearchEngine, DeviceHashScorer, _, LseRecorder = _pkg()
    vocab = P.Vocabulary(V, 0, 2)
    cfg = P.DecodeConfig(k=k, n=n, epsilon=1 / 6, delta=3.0, max_candidates=4, max_len=12)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(5, Nin, V, mean_len=6.0, clip=20))
    rec = LseRecorder(DeviceHashScorer(vocab, 11, scale=scale, power=power, eos_bias=eb, dtype=dt),
                      record_logits=True)
    P.run_varstream(corpus, rec, cfg)
    cpu = HashLogitsCPU(V, 0, 2, 11, scale=scale, power=power, eos_bias=eb, dtype=dt)
    assert len(rec.logit_table) > 4 * n
    for (iid, toks), got in rec.logit_table.items():
        want = cpu.logits(cpu.encode(corpus[iid], iid), toks)
        assert np.array_equal(got.view(np.uint32), want.astype(np.float32).view(np.uint32)), (iid, toks)


# The bench's own workloads (bench.py WORKLOADS) at their exact engine shapes:
# name, V, k, n, M, delta, max_len, N (a prefix of the bench's corpus
# generator: geometric, seed 99), mean_len, clip, scorer seed, scale, eos_bias
BENCH_SHAPES = [
    ("wmt19_k50", 42024, 50, 128, 5, 1.5, 256, 320, 25.0, 200, 7, 0.5, 7.5),
    ("parse_c3", 2048, 10, 256, 3, 10.0, 64, 1200, 12.0, None, 5, 0.5, 5.5),
]


@pytest.mark.parametrize("shape", BENCH_SHAPES, ids=[b[0] for b in BENCH_SHAPES])
def test_bench_shape_decode_bit_exact_vs_oracle(shape):
    """SURVEY §8(a) at the bench's exact engine shapes (C4: |V|=42,024, k=50,
    n=128, M=5, δ=1.5; C3: |V|=2,048, k=10, n=256, M=3, δ=10), with enough
    inputs that the ε-refill runs many times: every StepEvent, output token and
    fp64 score bit-exact vs the oracle replaying the kernel's lse; the sync-free
    graphed driver and the bench's 4 concurrent batches give the same outputs."""
    name, V, k, n, M, delta, ml, Nin, mean, clip, seed, scale, eb = shape
    P, N, SearchEngine, DeviceHashScorer, _, LseRecorder = _pkg()
    vocab = P.Vocabulary(V, 0, 2)
    cfg = P.DecodeConfig(k=k, n=n, epsilon=1 / 6, delta=delta, max_candidates=M, max_len=ml)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(99, Nin, V, mean_len=mean, clip=clip))
    sc = DeviceHashScorer(vocab, seed, scale=scale, power=0, eos_bias=eb, dtype="bf16")
    rec = LseRecorder(sc)
    ev = []
    out, rep = P.run_varstream(corpus, rec, cfg, trace=True, on_step=ev.append)
    refills = sum(1 for e in ev if e.refilled)
    assert refills >= 3, "the refill path was not exercised"
    cpu = LseReplayScorer(HashLogitsCPU(V, 0, 2, seed, scale=scale, power=0, eos_bias=eb,
                                        dtype="bf16"), rec.table)
    oev = []
    want, wrep = O.run_varstream(corpus, cpu, O.as_oconfig(cfg), trace=True, on_step=oev.append)
    assert _events(ev) == _events(oev)
    sig = O.signature(want)
    assert [[(c.tokens, c.score) for c in per] for per in out] == sig
    assert rep.candidate_expansions == wrep.candidate_expansions
    fast, frep = P.run_varstream(corpus, sc, cfg)
    assert [[(c.tokens, c.score) for c in per] for per in fast] == sig
    assert frep.candidate_expansions == wrep.candidate_expansions
    many, _ = P.run_varstream(corpus, sc, cfg, streams=4)
    assert [[(c.tokens, c.score) for c in per] for per in many] == sig


def test_epsilon_and_scheduler_invariance_on_device():
    """SPEC exactness/ε-independence (bb SPEC.md:379-380): outputs and expansion
    totals identical across ε and across varstream/varbeam/varfifo."""
    P, N, SearchEngine, DeviceHashScorer, *_ = _pkg()
    vocab = P.Vocabulary(1000, 0, 2)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(4242, 300, 1000, mean_len=8.0))
    sig = None
    for runner, eps in ((P.run_varstream, 1 / 12), (P.run_varstream, 1 / 6), (P.run_varstream, 1 / 4),
                        (P.run_varbeam, 1 / 6), (P.run_varfifo, 1 / 6)):
        cfg = P.DecodeConfig(k=5, n=16, epsilon=eps, delta=1.5, max_candidates=3, max_len=48)
        out, rep = runner(corpus, DeviceHashScorer(vocab, 31337, eos_bias=6.0), cfg)
        s = ([[(c.tokens, c.score) for c in per] for per in out], rep.candidate_expansions)
        sig = sig or s
        assert s == sig


def test_rows_copy_kernel():
    P, N, *_ = _pkg()
    lib = N.load_library()
    planes, rows, maxpos, d = 3, 10, 6, 8
    buf = torch.arange(planes * rows * maxpos * d, dtype=torch.float32, device="cuda").view(
        planes, rows, maxpos, d)
    ref = buf.clone()
    cl = torch.tensor([1, 4, 3, 2, 7, 5], dtype=torch.int32, device="cuda")
    nc = torch.tensor([2], dtype=torch.int32, device="cuda")
    rc = lib.vs_rows_copy(buf.data_ptr(), buf.stride(0) * 4, planes, buf.stride(1) * 4, d * 4,
                          cl.data_ptr(), nc.data_ptr(), 4, torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    ref[:, 4, :3] = ref[:, 1, :3]
    ref[:, 7, :5] = ref[:, 2, :5]
    assert torch.equal(buf, ref)


def _toy_decoder_run(policy_runner="run_varstream"):
    P, N, SearchEngine, _, _, LseRecorder = _pkg()
    from paper_2010_02164_b200.decoder import TransformerScorer

    vocab = P.Vocabulary(300, 0, 2)
    cfg = P.DecodeConfig(k=5, n=8, epsilon=1 / 4, delta=2.5, max_candidates=3, max_len=20)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(11, 40, 300, mean_len=6.0, clip=30))
    dec = TransformerScorer(vocab, d=32, heads=4, layers=2, enc_layers=1, ffn=64, max_src=32, seed=3,
                            tau=3.0, eos_bias=3.0, record_logits=True)
    rec = LseRecorder(dec, record_logits=True)
    ev = []
    out, rep = getattr(P, policy_runner)(corpus, rec, cfg, trace=True, on_step=ev.append)
    return P, vocab, cfg, corpus, dec, rec, ev, out, rep


def test_decoder_kv_cache_with_k4_reorder_matches_full_recompute():
    """Incremental decoding through the physical-row K/V cache, reordered by
    K4 from K2's copy plan, reproduces a cache-free forward of every sampled
    prefix (fp32, tolerance 2e-4)."""
    P, vocab, cfg, corpus, dec, rec, ev, out, rep = _toy_decoder_run()
    assert dec.copies > 0, "no K4 copies exercised"
    keys = sorted(rec.logit_table)
    rng = np.random.default_rng(0)
    sample = [keys[i] for i in rng.choice(len(keys), size=min(60, len(keys)), replace=False)]
    # prefer long prefixes (more reorders upstream)
    sample += sorted(keys, key=lambda kk: -len(kk[1]))[:20]
    for iid, toks in sample:
        want = dec.full_forward(corpus[iid], toks).cpu().numpy()
        got = rec.logit_table[(iid, toks)]
        assert np.max(np.abs(got - want)) < 2e-4, (iid, toks)


def test_decoder_decisions_match_oracle_replay():
    """Every search decision on decoder logits is bit-exact vs the oracle
    replaying the recorded rows (logits, kernel lse)."""
    from oracle.scorers import RecordedRowsScorer

    P, vocab, cfg, corpus, dec, rec, ev, out, rep = _toy_decoder_run()
    cpu = RecordedRowsScorer(vocab.size, vocab.sos, vocab.eos, rec.logit_table, rec.table)
    oev = []
    want, wrep = O.run_varstream(corpus, cpu, O.as_oconfig(cfg), trace=True, on_step=oev.append)
    assert _events(ev) == _events(oev)
    assert [[(c.tokens, c.score) for c in per] for per in out] == O.signature(want)


def _graphed_decoder_run(use_graphs=True, fused_head=False):
    P, N, SearchEngine, _, _, LseRecorder = _pkg()
    from paper_2010_02164_b200.decoder import GraphedTransformerScorer

    vocab = P.Vocabulary(500, 0, 2)
    cfg = P.DecodeConfig(k=6, n=8, epsilon=1 / 4, delta=2.0, max_candidates=3, max_len=24)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(5, 40, 500, mean_len=7.0, clip=30))
    dec = GraphedTransformerScorer(vocab, d=256, heads=4, layers=2, enc_layers=1, ffn=512, max_src=32,
                                   seed=4, tau=3.0, eos_bias=4.0, use_graphs=use_graphs, fused_head=fused_head)
    rec = LseRecorder(dec, record_logits=True)
    ev = []
    out, rep = P.run_varstream(corpus, rec, cfg, trace=True, on_step=ev.append)
    return P, vocab, cfg, corpus, dec, rec, ev, out, rep


def test_graphed_decoder_matches_cache_free_forward():
    """The WMT-shape scorer path (bf16, vs_row_attention in place over the
    physical-row cache with fused append, K4 reorders, CUDA-graph replay per
    row bucket) reproduces a cache-free bf16 forward of sampled prefixes
    (bf16 model: tolerance 0.06 + 2% of the logit scale)."""
    P, vocab, cfg, corpus, dec, rec, ev, out, rep = _graphed_decoder_run()
    assert len(dec.graphs) >= 1
    keys = sorted(rec.logit_table)
    rng = np.random.default_rng(1)
    sample = [keys[i] for i in rng.choice(len(keys), size=min(40, len(keys)), replace=False)]
    sample += sorted(keys, key=lambda kk: -len(kk[1]))[:10]
    worst = 0.0
    for iid, toks in sample:
        want = dec.full_forward(corpus[iid], toks).cpu().numpy()
        got = rec.logit_table[(iid, toks)]
        err = float(np.max(np.abs(got - want)))
        worst = max(worst, err / (0.06 + 0.02 * float(np.max(np.abs(want)))))
    assert worst <= 1.0, worst


def test_graphed_decoder_decisions_match_oracle_replay_and_eager():
    """Decisions on the graphed decoder's logits are bit-exact vs the oracle
    replaying the recorded rows; graph replay and eager execution of the same
    step body give identical outputs."""
    from oracle.scorers import RecordedRowsScorer

    P, vocab, cfg, corpus, dec, rec, ev, out, rep = _graphed_decoder_run()
    cpu = RecordedRowsScorer(vocab.size, vocab.sos, vocab.eos, rec.logit_table, rec.table)
    oev = []
    want, wrep = O.run_varstream(corpus, cpu, O.as_oconfig(cfg), trace=True, on_step=oev.append)
    assert _events(ev) == _events(oev)
    assert [[(c.tokens, c.score) for c in per] for per in out] == O.signature(want)
    *_, out2, rep2 = _graphed_decoder_run(use_graphs=False)
    assert [[(c.tokens, c.score) for c in per] for per in out2] == [[(c.tokens, c.score) for c in per] for per in out]


@pytest.mark.parametrize("R,V,M", [(1, 1000, 5), (37, 5003, 5), (300, 42024, 5), (129, 2048, 8)])
def test_proj_topm_tcgen05_matches_oracle(R, V, M):
    """K5: tcgen05 vocab projection with the fused K1 epilogue.  Its bf16
    logits match a torch fp32 GEMM within one bf16 ulp (different accumulation
    order), and every top-M decision/logp is bit-exact vs the oracle on the
    logits it wrote (K1's contract), with lse within 1e-5 of fp64."""
    from paper_2010_02164_b200.search import proj_lse_topm

    torch.manual_seed(R + V)
    K = 1024
    h = (torch.randn(R, K, device="cuda") * 0.5).to(torch.bfloat16)
    w = (torch.randn(V, K, device="cuda") / 16).to(torch.bfloat16)
    eos = 2
    eos_add = torch.rand(R, device="cuda") * 3
    tok, lp, lse, fb, lg = proj_lse_topm(h, w, M, eos=eos, eos_add=eos_add)
    torch.cuda.synchronize()
    ref = (h.float() @ w.float().T)
    ref_bf = ref.to(torch.bfloat16).float()
    ref_bf[:, eos] = (ref_bf[:, eos] + eos_add).to(torch.bfloat16).float()
    got = lg.float()
    ulp = ref_bf.abs().clamp_min(1e-3) * 2.0 ** -7
    assert bool(((got - ref_bf).abs() <= ulp + 1e-6).all()), float((got - ref_bf).abs().max())
    x = got.cpu().numpy()
    _check_rows(x, M, tok.cpu().numpy(), lp.cpu().numpy(), lse.cpu().numpy())


def test_graphed_decoder_with_fused_k5_head_matches_oracle_replay():
    """The decoder with the tcgen05 vocab projection + fused K1 (K5) inside the
    step graph: every decision bit-exact vs the oracle replaying the logits K5
    wrote and the lse it exported; logits match the cache-free forward."""
    from oracle.scorers import RecordedRowsScorer

    P, vocab, cfg, corpus, dec, rec, ev, out, rep = _graphed_decoder_run(fused_head=True)
    cpu = RecordedRowsScorer(vocab.size, vocab.sos, vocab.eos, rec.logit_table, rec.table)
    oev = []
    want, wrep = O.run_varstream(corpus, cpu, O.as_oconfig(cfg), trace=True, on_step=oev.append)
    assert _events(ev) == _events(oev)
    assert [[(c.tokens, c.score) for c in per] for per in out] == O.signature(want)
    keys = sorted(rec.logit_table)
    for iid, toks in keys[:: max(1, len(keys) // 30)]:
        want_l = dec.full_forward(corpus[iid], toks).cpu().numpy()
        got = rec.logit_table[(iid, toks)]
        assert np.max(np.abs(got - want_l)) <= 0.06 + 0.02 * float(np.max(np.abs(want_l)))


def test_concurrent_batches_match_single_batch():
    """run_varstream(streams=3): three refilling batches driven concurrently on
    separate CUDA streams produce exactly the single-batch candidates."""
    P, N, SearchEngine, DeviceHashScorer, _, _ = _pkg()
    vocab = P.Vocabulary(5000, 0, 2)
    cfg = P.DecodeConfig(k=8, n=16, epsilon=1 / 6, delta=1.5, max_candidates=3, max_len=40)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(3, 300, 5000, mean_len=9.0, clip=30))
    sc = DeviceHashScorer(vocab, 17, scale=0.5, power=0, eos_bias=5.0, dtype="bf16")
    one, rep1 = P.run_varstream(corpus, sc, cfg)
    many, rep3 = P.run_varstream(corpus, sc.fork(), cfg, streams=3)
    assert [[(c.tokens, c.score) for c in per] for per in many] == [[(c.tokens, c.score) for c in per] for per in one]


def test_repeated_calls_reuse_engine_and_graphs_correctly():
    """The public API reuses engines, buffers and captured step graphs across
    calls: corpora of different sizes (larger, smaller, same) in sequence, on
    1 and 3 concurrent batches, each give exactly the synchronous driver's
    candidates (that path is checked against the oracle above).  A stale graph
    (e.g. the K3 input-count argument) would show up here."""
    P, N, SearchEngine, DeviceHashScorer, _, LseRecorder = _pkg()
    from oracle.scorers import HashLogitsCPU, LseReplayScorer

    vocab = P.Vocabulary(3000, 0, 2)
    cfg = P.DecodeConfig(k=6, n=12, epsilon=1 / 6, delta=1.5, max_candidates=3, max_len=30)
    sc = DeviceHashScorer(vocab, 23, scale=0.5, power=0, eos_bias=5.0, dtype="bf16")
    for seed, n_in in [(1, 90), (2, 140), (3, 40), (4, 140)]:
        corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(seed, n_in, 3000, mean_len=8.0, clip=25))
        ref_out, _ = P.run_varstream(corpus, LseRecorder(sc), cfg)  # sync driver: exports lse
        fast, _ = P.run_varstream(corpus, sc, cfg)
        many, _ = P.run_varstream(corpus, sc, cfg, streams=3)
        sig = [[(c.tokens, c.score) for c in per] for per in ref_out]
        assert [[(c.tokens, c.score) for c in per] for per in fast] == sig
        assert [[(c.tokens, c.score) for c in per] for per in many] == sig


def _sharded_worker(rank, world, port, out_path):
    import os
    import pickle

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2010_02164_b200 as P
    from paper_2010_02164_b200.parallel import run_varstream_sharded
    from paper_2010_02164_b200.scorers import DeviceHashScorer

    vocab = P.Vocabulary(3000, 0, 2)
    cfg = P.DecodeConfig(k=6, n=12, epsilon=1 / 6, delta=1.5, max_candidates=3, max_len=30)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(9, 150, 3000, mean_len=8.0, clip=25))
    sc = DeviceHashScorer(vocab, 29, scale=0.5, power=0, eos_bias=5.0, dtype="bf16")
    res, _ = run_varstream_sharded(corpus, sc, cfg, streams=2)
    if rank == 0:
        with open(out_path, "wb") as f:
            pickle.dump([[(c.tokens, c.score) for c in per] for per in res], f)
    dist.destroy_process_group()


def test_sharded_concurrent_run_gathers_single_run_outputs(tmp_path):
    """Two ranks (gloo, sharing this GPU), each running 2 concurrent batches:
    rank 0's gathered outputs equal a single-process, single-batch decode."""
    import pickle
    import socket

    import torch.multiprocessing as mp

    P, N, SearchEngine, DeviceHashScorer, _, _ = _pkg()
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    out = tmp_path / "sharded.pkl"
    mp.spawn(_sharded_worker, args=(2, port, str(out)), nprocs=2, join=True)
    vocab = P.Vocabulary(3000, 0, 2)
    cfg = P.DecodeConfig(k=6, n=12, epsilon=1 / 6, delta=1.5, max_candidates=3, max_len=30)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(9, 150, 3000, mean_len=8.0, clip=25))
    sc = DeviceHashScorer(vocab, 29, scale=0.5, power=0, eos_bias=5.0, dtype="bf16")
    want, _ = P.run_varstream(corpus, sc, cfg)
    got = pickle.loads(out.read_bytes())
    assert got == [[(c.tokens, c.score) for c in per] for per in want]


@pytest.mark.parametrize("append", [False, True])
def test_row_attention_matches_torch(append):
    """vs_row_attention (in-place decode attention over cache rows, optional
    append of the newest position) and vs_row_attention_grouped (rows sharing a
    cache row, tensor-core tiles; groups of 1..70 rows, 1..256 positions) vs a
    torch fp32 softmax attention."""
    P, N, *_ = _pkg()
    lib = N.load_library()
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(7)
    H, D, nrow, Lmax = 8, 64, 6, 256
    lens_g = [1, 5, 33, 64, 200, 256]  # per cache row
    groups = [(0, 3), (1, 2), (2, 7), (3, 1), (4, 70), (5, 2)]  # (cache row, rows in group)
    idx = torch.tensor([c for c, n_ in groups for _ in range(n_)], dtype=torch.int32, device=dev)
    lens = torch.tensor([lens_g[c] for c, n_ in groups for _ in range(n_)], dtype=torch.int32, device=dev)
    R = idx.numel()
    kc = torch.randn(nrow, Lmax, H * D, generator=g, device=dev).to(torch.bfloat16)
    vc = torch.randn(nrow, Lmax, H * D, generator=g, device=dev).to(torch.bfloat16)
    q = torch.randn(R, H * D, generator=g, device=dev).to(torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    out = torch.empty(R, H * D, dtype=torch.bfloat16, device=dev)
    if append:  # one private cache row per query row, newest position from k_new/v_new
        rows = torch.arange(R, dtype=torch.int32, device=dev)
        kc2 = kc[idx.long()].clone()
        vc2 = vc[idx.long()].clone()
        kn = torch.randn(R, H * D, generator=g, device=dev).to(torch.bfloat16)
        vn = torch.randn(R, H * D, generator=g, device=dev).to(torch.bfloat16)
        N.check(lib.vs_row_attention(q.data_ptr(), q.stride(0), kc2.data_ptr(), vc2.data_ptr(), kc2.stride(0),
                                     kc2.stride(1), rows.data_ptr(), lens.data_ptr(), kn.data_ptr(), vn.data_ptr(),
                                     kn.stride(0), out.data_ptr(), out.stride(0), H, D, 0.125, R, None, R, st),
                "attn")
        ar = torch.arange(R, device=dev)
        assert torch.equal(kc2[ar, lens.long() - 1], kn) and torch.equal(vc2[ar, lens.long() - 1], vn)
        K, Vv = kc2, vc2
        crow = ar
    else:
        N.check(lib.vs_row_attention(q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(), kc.stride(0),
                                     kc.stride(1), idx.data_ptr(), lens.data_ptr(), None, None, 0, out.data_ptr(),
                                     out.stride(0), H, D, 0.125, R, None, R, st), "attn")
        K, Vv = kc, vc
        crow = idx.long()
    torch.cuda.synchronize()
    refs = []
    for r in range(R):
        L = int(lens[r])
        qq = q[r].float().view(H, D)
        kk = K[crow[r], :L].float().view(L, H, D)
        vv = Vv[crow[r], :L].float().view(L, H, D)
        p = torch.softmax(torch.einsum("hd,lhd->hl", qq, kk) * 0.125, dim=-1)
        refs.append(torch.einsum("hl,lhd->hd", p, vv).reshape(-1))
        assert torch.allclose(out[r].float(), refs[-1], atol=2e-2, rtol=2e-2), f"row {r}"
    if not append:
        off = torch.tensor(np.concatenate([[0], np.cumsum([n_ for _, n_ in groups])]), dtype=torch.int32,
                           device=dev)
        ng = torch.tensor([len(groups)], dtype=torch.int32, device=dev)
        out2 = torch.full_like(out, float("nan"))
        N.check(lib.vs_row_attention_grouped(q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(), kc.stride(0),
                                             kc.stride(1), idx.data_ptr(), lens.data_ptr(), off.data_ptr(),
                                             ng.data_ptr(), len(groups) + 2, out2.data_ptr(), out2.stride(0), H, D,
                                             0.125, st), "attn_grouped")
        torch.cuda.synchronize()
        for r in range(R):
            assert torch.allclose(out2[r].float(), refs[r], atol=2e-2, rtol=2e-2), f"grouped row {r}"


def test_end_to_end_agreement_with_fp64_reference_rows():
    """north_star: decoded outputs match the reference algorithm computing its
    OWN fp64 log-softmax rows (no lse replay) on the same logits on >= 99.5% of
    inputs, every score within 1e-5 relative."""
    P, N, SearchEngine, DeviceHashScorer, _, _ = _pkg()
    V = 6000
    vocab = P.Vocabulary(V, 0, 2)
    cfg = P.DecodeConfig(k=12, n=24, epsilon=1 / 6, delta=1.5, max_candidates=4, max_len=40)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(77, 240, V, mean_len=10.0, clip=30))
    sc = DeviceHashScorer(vocab, 4242, scale=0.5, power=0, eos_bias=6.0, dtype="bf16")
    got, _ = P.run_varstream(corpus, sc, cfg, streams=2)
    cpu = HashLogitsCPU(V, vocab.sos, vocab.eos, 4242, scale=0.5, power=0, eos_bias=6.0, dtype="bf16")
    want, _ = O.run_varstream(corpus, cpu, O.as_oconfig(cfg))
    same, worst = 0, 0.0
    for g_, w_ in zip(got, want):
        ok = len(g_) == len(w_) and all(tuple(a.tokens) == tuple(b.tokens) for a, b in zip(g_, w_))
        if ok:
            rel = max(abs(a.score - b.score) / max(1e-12, abs(b.score)) for a, b in zip(g_, w_))
            worst = max(worst, rel)
            ok = rel <= 1e-5
        same += ok
    assert same / len(corpus) >= 0.995, (same, len(corpus))
    assert worst <= 1e-5


def test_decoder_end_to_end_agreement_with_reference_search():
    """north_star's decoder-path agreement: the device engine driving the
    transformer decoder (fp32, physical-row K/V cache + K4, row kernels) vs
    the REFERENCE search (oracle restatement of bb/scheduler.py run_varstream)
    driving the same random-init model on the CPU through the stateless
    Scorer protocol (oracle/scorers.py:TorchDecoderCPU, whole-prefix
    recompute, fp64 log-softmax rows).  >= 99.5% of inputs identical (tokens
    equal, scores within 1e-5 relative); every divergence is an fp near-tie:
    the reference itself decided it by a margin <= 1e-4 (oracle/agreement.py)."""
    from oracle.agreement import agreement_report
    from oracle.scorers import TorchDecoderCPU
    from paper_2010_02164_b200.decoder import TransformerScorer

    P, *_ = _pkg()
    V = 500
    kw = dict(d=64, heads=4, layers=2, enc_layers=1, ffn=128, seed=3, tau=4.0)
    vocab = P.Vocabulary(V, 0, 2)
    cfg = P.DecodeConfig(k=5, n=16, epsilon=1 / 6, delta=2.5, max_candidates=3, max_len=24)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(21, 200, V, mean_len=6.0, clip=30))
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        dec = TransformerScorer(vocab, max_src=32, eos_bias=4.0, dtype=torch.float32, **kw)
        out, rep = P.run_varstream(corpus, dec, cfg)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    cpu = TorchDecoderCPU(V, 0, 2, eos_bias=4.0, weights="f32", **kw)
    want, wrep = O.run_varstream(corpus, cpu, O.as_oconfig(cfg))
    ids = list(range(len(corpus)))
    gsig = {i: [(c.tokens, c.score) for c in out[i]] for i in ids}
    csig = dict(enumerate(O.signature(want)))
    r = agreement_report(corpus, ids, gsig, csig, cpu, O.as_oconfig(cfg), tie_tol=1e-4)
    assert r["identical_fraction"] >= 0.995, r
    assert r["explained_by_near_ties"] == r["divergent"], r


def test_api_per_beam_and_batch_pieces_reproduce_reference():
    """The reference's own driver loop (bb/scheduler.py:243-287) written with
    this package's API pieces — refill, select_min_lt, execute_step (all
    selected beams expanded in one device step), flush_all — plus
    beam_decode / greedy_decode per input, on the reference scorer: events,
    outputs and fp64 scores equal the oracle's (pinned to the reference)."""
    import math as _m

    P, *_ = _pkg()
    from paper_2010_02164_b200 import api as A

    fx = RUNS["c1_varstream_flush7"]
    s = fx["scorer"]
    base = SeededHashScorerCPU(s["vocab_size"], s["sos"], s["eos"], s["seed"], s["eos_bias"])
    vocab = P.Vocabulary(s["vocab_size"], s["sos"], s["eos"])
    sc = _RefVocabScorer(base, vocab)
    d = fx["config"]
    cfg = P.DecodeConfig(k=d["k"], n=d["n"], epsilon=d["epsilon"], delta=fl(d["delta"]),
                         max_candidates=d["max_candidates"], max_len=d["max_len"],
                         flush_interval=d["flush_interval"])
    corpus = [tuple(x) for x in fx["corpus"]][:70]
    ev = []
    state, rep = A.BatchState(), P.MetricsReport.new(trace=True)
    thr = _m.floor(cfg.epsilon * cfg.n + 1e-9)
    next_flush = cfg.flush_interval
    while state.cursor < len(corpus) or state.beams:
        if state.timestep >= next_flush:
            if state.beams:
                A.flush_all(state, sc, cfg, rep, ev.append)
            next_flush = state.timestep + cfg.flush_interval
        refilled = A.refill(state, corpus, cfg, sc) if len(state.beams) <= thr else []
        if not state.beams:
            break
        A.execute_step(state, A.select_min_lt(state, cfg.capacity), sc, cfg, rep, refilled=refilled,
                       on_step=ev.append)
    out = [state.outputs[i] for i in range(len(corpus))]
    oev = []
    want, wrep = O.run_varstream(corpus, base, O.as_oconfig(cfg), trace=True, on_step=oev.append)
    assert _events(ev) == _events(oev)
    assert [[(c.tokens, c.score) for c in per] for per in out] == O.signature(want)
    assert [tuple(r) for r in rep.per_step_trace] == [tuple(r) for r in wrep.per_step_trace]
    for i in range(0, 70, 7):  # the unbatched reference per input, and greedy
        enc = base.encode(corpus[i], i)
        assert [(c.tokens, c.score) for c in A.beam_decode(enc, sc, cfg)] == O.signature([want[i]])[0]
        g = A.greedy_decode(enc, sc, cfg.max_len)
        og = O.greedy_decode(enc, base, cfg.max_len)
        assert (g.tokens, g.score) == (og.tokens, og.score)


def _lstm_run(use_graphs=True, k=6, n=8, N_in=48):
    P, N, SearchEngine, _, _, LseRecorder = _pkg()
    from paper_2010_02164_b200.decoder import LSTMScorer

    vocab = P.Vocabulary(700, 0, 2)
    cfg = P.DecodeConfig(k=k, n=n, epsilon=1 / 4, delta=3.0, max_candidates=3, max_len=20)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(8, N_in, 700, mean_len=7.0, clip=40))
    dec = LSTMScorer(vocab, emb=64, hidden=256, max_src=64, seed=2, tau=3.0, eos_bias=4.0, use_graphs=use_graphs)
    rec = LseRecorder(dec, record_logits=True)
    ev = []
    out, rep = P.run_varstream(corpus, rec, cfg, trace=True, on_step=ev.append)
    return P, vocab, cfg, corpus, dec, rec, ev, out, rep


def test_lstm_scorer_state_reorder_matches_full_recompute():
    """configs[2]'s LSTM decoder: the per-physical-row (h, c) state, moved by
    K4 in fixed-size mode from K2's copy plan, and the grouped tensor-core
    attention over the slot's encoder states reproduce a cache-free forward
    of sampled prefixes (bf16 operands: tolerance 0.05 + 2% of the scale)."""
    P, vocab, cfg, corpus, dec, rec, ev, out, rep = _lstm_run()
    keys = sorted(rec.logit_table)
    rng = np.random.default_rng(3)
    sample = [keys[i] for i in rng.choice(len(keys), size=min(40, len(keys)), replace=False)]
    sample += sorted(keys, key=lambda kk: -len(kk[1]))[:10]
    worst = 0.0
    for iid, toks in sample:
        want = dec.full_forward(corpus[iid], toks).cpu().numpy()
        got = rec.logit_table[(iid, toks)]
        worst = max(worst, float(np.max(np.abs(got - want))) / (0.05 + 0.02 * float(np.max(np.abs(want)))))
    assert worst <= 1.0, worst


def test_lstm_scorer_decisions_match_oracle_replay_and_eager():
    from oracle.scorers import RecordedRowsScorer

    P, vocab, cfg, corpus, dec, rec, ev, out, rep = _lstm_run()
    assert len(dec.graphs) >= 1
    cpu = RecordedRowsScorer(vocab.size, vocab.sos, vocab.eos, rec.logit_table, rec.table)
    oev = []
    want, wrep = O.run_varstream(corpus, cpu, O.as_oconfig(cfg), trace=True, on_step=oev.append)
    assert _events(ev) == _events(oev)
    assert [[(c.tokens, c.score) for c in per] for per in out] == O.signature(want)
    *_, out2, rep2 = _lstm_run(use_graphs=False)
    assert [[(c.tokens, c.score) for c in per] for per in out2] == [[(c.tokens, c.score) for c in per] for per in out]


@pytest.mark.parametrize("M", [1, 5, 8, 32])
def test_row_topm_split_rows_with_concentrated_and_tied_maxima(M):
    """Small steps run several warps per row whose bootstrap θ is pooled across
    the row's parts: rows whose largest values all sit in one part, rows made of
    ties, and a row whose maximum is in the scalar tail stay exact (warp kernel
    and split kernel)."""
    P, *_ = _pkg()
    V = 42023  # odd: a scalar tail
    rng = np.random.default_rng(17)
    x = rng.normal(0, 1, (4, V)).astype(np.float32)
    x[0, 40000:40040] += 9.0          # the top region inside the last part
    x[1, :] = 0.5                       # all tied
    x[1, 7::997] = 0.75
    x[2, V - 1] = 50.0                  # maximum in the tail
    x[3, :] = np.round(x[3, :], 1)     # heavy ties
    for dt in (torch.float32, torch.bfloat16):
        dx = torch.from_numpy(x).cuda().to(dt)
        for kernel in ("warp", "split"):
            tok, lp, lse, _ = P.row_lse_topm(dx, M, kernel=kernel)
            _check_rows(dx.float().cpu().numpy(), M, tok.cpu().numpy(), lp.cpu().numpy(), lse.cpu().numpy())


@pytest.mark.parametrize("d", [256, 1024])
def test_layer_norm_kernel_matches_torch(d):
    """vs_layer_norm_bf16 (decoder LayerNorm) vs F.layer_norm on bf16 rows:
    within one bf16 ulp of the fp32 result."""
    P, N, *_ = _pkg()
    lib = N.load_library()
    g = torch.Generator(device="cuda").manual_seed(d)
    x = (torch.randn((333, d), generator=g, device="cuda") * 3 + 1.5).to(torch.bfloat16)
    y = torch.empty_like(x)
    N.check(lib.vs_layer_norm_bf16(x.data_ptr(), x.stride(0), y.data_ptr(), y.stride(0), x.shape[0], d, 1e-5,
                                   torch.cuda.current_stream().cuda_stream), "ln")
    torch.cuda.synchronize()
    ref = torch.nn.functional.layer_norm(x.float(), (d,))
    assert torch.allclose(y.float(), ref, rtol=1e-2, atol=1e-2)
    assert (y.float() - torch.nn.functional.layer_norm(x, (d,)).float()).abs().max() <= 0.02


def _nccl_worker(rank, world, port, out_path):
    import os
    import pickle

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda:0"))
    import paper_2010_02164_b200 as P
    from paper_2010_02164_b200.parallel import run_varstream_sharded
    from paper_2010_02164_b200.scorers import DeviceHashScorer

    vocab = P.Vocabulary(3000, 0, 2)
    cfg = P.DecodeConfig(k=6, n=12, epsilon=1 / 6, delta=1.5, max_candidates=3, max_len=30)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(9, 150, 3000, mean_len=8.0, clip=25))
    sc = DeviceHashScorer(vocab, 29, scale=0.5, power=0, eos_bias=5.0, dtype="bf16")
    res, _ = run_varstream_sharded(corpus, sc, cfg, streams=2)
    with open(out_path, "wb") as f:
        pickle.dump([[(c.tokens, c.score) for c in per] for per in res], f)
    dist.destroy_process_group()


def test_nccl_gather_path_single_rank(tmp_path):
    """The multi-GPU data plane over NCCL (one rank on this GPU: the all-reduce
    of the message size and the gather of the packed message run through
    ProcessGroupNCCL) returns the single-process outputs."""
    import pickle
    import socket

    import torch.multiprocessing as mp

    P, N, SearchEngine, DeviceHashScorer, _, _ = _pkg()
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    out = tmp_path / "nccl.pkl"
    mp.spawn(_nccl_worker, args=(1, port, str(out)), nprocs=1, join=True)
    vocab = P.Vocabulary(3000, 0, 2)
    cfg = P.DecodeConfig(k=6, n=12, epsilon=1 / 6, delta=1.5, max_candidates=3, max_len=30)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(9, 150, 3000, mean_len=8.0, clip=25))
    sc = DeviceHashScorer(vocab, 29, scale=0.5, power=0, eos_bias=5.0, dtype="bf16")
    want, _ = P.run_varstream(corpus, sc, cfg)
    assert pickle.loads(out.read_bytes()) == [[(c.tokens, c.score) for c in per] for per in want]


@pytest.mark.parametrize("chunk", [1, 7, 10 ** 9])
def test_streamed_output_harvest_matches_synchronous_results(chunk):
    """Harvest: outputs copied and materialised while the device decodes
    (chunks of finished inputs below MINLIVE, appended token ranges below
    TOKFILL) equal the synchronous driver's results for any chunk size."""
    P, N, SearchEngine, DeviceHashScorer, _, _ = _pkg()
    vocab = P.Vocabulary(2000, 0, 2)
    cfg = P.DecodeConfig(k=7, n=10, epsilon=1 / 5, delta=1.5, max_candidates=3, max_len=28)
    corpus, _ = O.bucket_by_length(O.generate_synthetic_corpus(12, 130, 2000, mean_len=7.0, clip=20))
    sc = DeviceHashScorer(vocab, 41, scale=0.5, power=0, eos_bias=4.0, dtype="bf16")
    want, wrep = SearchEngine(cfg, vocab).run(corpus, sc, admit_mode=N.VS_ADMIT_VARSTREAM,
                                              select_mode=N.VS_SELECT_MIN_LT, flush_enabled=False)
    eng = SearchEngine(cfg, vocab)
    out = [[] for _ in range(len(corpus))]
    gen = eng.async_steps(corpus, sc, admit_mode=N.VS_ADMIT_VARSTREAM, select_mode=N.VS_SELECT_MIN_LT,
                          harvest_into=out, harvest_chunk=chunk)
    for _ in gen:
        pass
    assert [[(c.tokens, c.score, c.input_id) for c in per] for per in out] == \
        [[(c.tokens, c.score, c.input_id) for c in per] for per in want]
    assert eng.last_d2h_bytes > 0


@pytest.mark.gpu
def test_device_path_rejects_bad_inputs_like_reference():
    """Empty inputs / out-of-vocabulary tokens raise the reference's DataErrors
    (bb/model.py:90-102) on the device path, before any kernel runs, for both
    the single-batch and the concurrent-batch drivers."""
    P, _, _, DeviceHashScorer, _, _ = _pkg()
    vocab = P.Vocabulary(16, 0, 2)
    cfg = P.DecodeConfig(k=2, n=2, epsilon=1 / 6, max_candidates=2, max_len=8)
    sc = DeviceHashScorer(vocab, 5)
    for streams in (1, 2):
        with pytest.raises(P.DataError, match="inputs must be nonempty"):
            P.run_varstream([[3, 4], [], [5]], sc, cfg, streams=streams)
        with pytest.raises(P.DataError, match=r"token 16 at position 2 is outside the vocabulary \(size 16\)"):
            P.run_varstream([[3, 4], [5, 6, 16], [5]], sc, cfg, streams=streams)
    out, _ = P.run_varstream([[3, 4], [5, 6, 7], [5]], sc, cfg)  # the engine is still usable
    assert len(out) == 3 and all(out)
