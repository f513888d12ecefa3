// K2 beam_step: per-beam merge, δ/M pruning, EOS finalisation, emission,
// length-cap drain and row planning (sm_100a).  One CTA (128 threads) per
// selected beam; every phase is data-parallel (no single-thread loops over
// candidates), so the critical path is a handful of barriers.
//
// Restates, for the deferred policy (bb/core.py:18-28):
//   _candidate_pool   bb/search.py:52-73   (no-ops + per-parent top-M, fp64 add)
//   apply_heuristics  bb/heuristics.py:81-93 (sort by bb/core.py:156-158 order,
//                     max_candidates_filter :42-64, absolute_threshold_filter :67-78)
//   _materialize/extend bb/search.py:106-117, bb/core.py:161-176
//   _expand_deferred  bb/search.py:120-145 (rank-1 finalized emission)
//   advance_beam      bb/search.py:215-230 + _drain_at_length_cap :190-202
//   beam_finished     bb/search.py:205-212
//
// Selection: the pool is w sorted lists (one per finalized candidate — its
// no-op — and one per active parent — its M proposals, K1's order re-checked
// against (score desc, token asc)).  An entry's rank is the sum over lists of
// how many of their entries precede it, counted from each list head; entries
// below kept[0].score - delta are never ranked.  The per-parent cap never
// binds (each parent contributes min(M, V) proposals, all accepted by
// max_candidates_filter), so kept = the first min(k, |pool|) entries at or
// above the δ cutoff.
//
// Row planning (new, no reference equivalent): candidates are logical; each
// owns a physical row of the slot (token history + scorer row state such as
// a KV cache).  The first child of a parent inherits the parent's row (no
// copy); further children take the rows left free, in ascending order, and
// get a (src,dst,len) copy entry.  Sources are always rows claimed by
// inheritors, destinations always free rows, so in-place copies are
// hazard-free.
#include <algorithm>

#include "schedule.cuh"

namespace vs {
namespace {

constexpr int NT2 = 128;  // == VS_MAX_K: one thread per candidate / child
constexpr unsigned FULLM = 0xffffffffu;

// Row value of top-M entry i: the exact fp64 row value when the rows were
// reference fp64 log-probs (vs_row_topm_f64), else K1's fp32 logp.
__device__ __forceinline__ double row_logp(const vs_state& st, int64_t i) {
  return st.top_logp64 ? st.top_logp64[i] : (double)st.top_logp[i];
}

struct Pool {
  const double* sc;
  const int* par;
  const int* tok;
  // entry f precedes e in proposal_order (score desc, parent asc, token asc)
  __device__ __forceinline__ bool before(int f, int e) const {
    const double a = sc[f], b = sc[e];
    if (a != b) return a > b;
    if (par[f] != par[e]) return par[f] < par[e];
    return tok[f] < tok[e];
  }
};

// Block-wide (NT2 threads) exclusive prefix count of a predicate.
__device__ __forceinline__ int block_prefix(bool pred, int* wsm, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(FULLM, pred);
  if (lane == 0) wsm[wid] = __popc(b);
  __syncthreads();
  int off = 0, tot = 0;
#pragma unroll
  for (int q = 0; q < NT2 / 32; ++q) {
    off += q < wid ? wsm[q] : 0;
    tot += wsm[q];
  }
  __syncthreads();
  *total = tot;
  return off + __popc(b & ((1u << lane) - 1u));
}

// Block-wide (NT2 threads) exclusive prefix sum of v.
__device__ __forceinline__ int block_prefix_sum(int v, int* wsm, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULLM, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsm[wid] = x;
  __syncthreads();
  int off = 0, tot = 0;
#pragma unroll
  for (int q = 0; q < NT2 / 32; ++q) {
    off += q < wid ? wsm[q] : 0;
    tot += wsm[q];
  }
  __syncthreads();
  *total = tot;
  return off + x - v;
}

__device__ __forceinline__ void beam_deferred(const vs_config& cfg, const vs_state& st, int M_rows,
                                              unsigned char* smem) {
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int k = cfg.k;
  // The beam's slot metadata and candidate state were written by launches that
  // completed before the top-M kernel now finishing (the one this launch
  // depends on) passed its own PDL wait, so they are loaded (from L2) under
  // that kernel's tail, before this CTA's wait; only the top-M outputs
  // (top_tok / top_logp / top_logp64) need the wait.
  const int s = __ldcg(&st.sel[b]);
  const int L = __ldcg(&st.slot_lt[s]);
  const int w = __ldcg(&st.slot_width[s]);
  const int row0 = __ldcg(&st.sel_off[b]);
  const int base = s * k;
  double p_sc = 0.0;
  unsigned long long p_h = 0;
  int p_l = 0, p_r = 0;
  bool isfin = false;
  if (tid < w) {
    p_sc = __ldcg(&st.c_score[base + tid]);
    p_h = __ldcg(reinterpret_cast<const unsigned long long*>(&st.c_hash[base + tid]));
    p_l = __ldcg(&st.c_len[base + tid]);
    p_r = __ldcg(&st.c_row[base + tid]);
    isfin = __ldcg(reinterpret_cast<const unsigned char*>(&st.c_fin[base + tid])) != 0;
  }
  VS_PDL_ENTRY();
  const int Meff = cfg.max_candidates < cfg.vocab_size ? cfg.max_candidates : cfg.vocab_size;
  const int Pmax = k + k * Meff;

  // ---- shared memory carve-up -------------------------------------------------
  double* cs = reinterpret_cast<double*>(smem);       // [k] current scores
  uint64_t* ch = reinterpret_cast<uint64_t*>(cs + k);  // [k] current hashes
  double* ps = reinterpret_cast<double*>(ch + k);     // [Pmax] pool score
  int* pp = reinterpret_cast<int*>(ps + Pmax);        // [Pmax] pool parent
  int* pt = pp + Pmax;                                // [Pmax] pool token (-1 = no-op)
  int* cl = pt + Pmax;                                // [k] current len
  int* cr = cl + k;                                   // [k] current row
  int* act = cr + k;                                  // [k] active ordinal -> cand idx
  int* fin = act + k;                                 // [k] finalized ordinal -> cand idx
  int* kept = fin + k;                                // [k] pool index by rank
  int* firstc = kept + k;                             // [k] first child of parent (atomicMin)
  int* claimed = firstc + k;                          // [k] row claimed
  int* freel = claimed + k;                           // [k] free rows, ascending
  int* emo = freel + k;                               // [k] emission order -> child
  int* nrow = emo + k;                                // [k] child row
  int* csrc = nrow + k;                               // [k] child copy source row (-1)
  int* nlen = csrc + k;                               // [k] child length
  int* ctok = nlen + k;                               // [k] child's new token (-1: no-op)
  int* prow = ctok + k;                               // [k] row holding the child's prefix
  int* eoff = prow + k;                               // [k] emission q's start in out_tok
  __shared__ int wsm[NT2 / 32];
  __shared__ int s_kept, s_nextra, s_ebase;
  __shared__ double s_cut;

  // ---- candidates -> smem; stable finalized / active split ---------------------
  if (tid < w) {
    cs[tid] = p_sc;
    ch[tid] = p_h;
    cl[tid] = p_l;
    cr[tid] = p_r;
  }
  if (tid < k) {
    firstc[tid] = 0x7fffffff;
    claimed[tid] = 0;
  }
  if (tid == 0) s_kept = 0;
  int nfz, nact;
  {
    const int fpos = block_prefix(tid < w && isfin, wsm, &nfz);
    const int apos = block_prefix(tid < w && !isfin, wsm, &nact);
    if (tid < w) {
      if (isfin) fin[fpos] = tid;
      else act[apos] = tid;
    }
  }
  __syncthreads();
  const int P = nfz + nact * Meff;

  VS_PROF(true, 1);
  // ---- pool (bb/search.py:64-72): no-ops, then per-parent top-M ----------------
  for (int e = tid; e < P; e += NT2) {
    if (e < nfz) {
      const int i = fin[e];
      ps[e] = cs[i];
      pp[e] = i;
      pt[e] = -1;
    } else {
      const int a = (e - nfz) / Meff, m = (e - nfz) - a * Meff;
      const int i = act[a];
      const int64_t ri = (int64_t)(row0 + a) * M_rows + m;
      ps[e] = cs[i] + row_logp(st, ri);  // fp64 add, bb/search.py:71
      pp[e] = i;
      pt[e] = st.top_tok[ri];
    }
  }
  __syncthreads();
  // per-parent lists sorted by (score desc, token asc); equal fp64 sums of
  // distinct logps may reorder K1's (logp desc, token asc) output (rare).
  for (int a = tid; a < nact; a += NT2) {
    const int b0 = nfz + a * Meff;
    bool sorted = true;
    for (int m = 0; m + 1 < Meff; ++m)
      if (ps[b0 + m] < ps[b0 + m + 1] || (ps[b0 + m] == ps[b0 + m + 1] && pt[b0 + m] > pt[b0 + m + 1]))
        sorted = false;
    if (!sorted)
      for (int m = 1; m < Meff; ++m) {
        const double sv = ps[b0 + m];
        const int tv = pt[b0 + m];
        int q = m - 1;
        while (q >= 0 && (ps[b0 + q] < sv || (ps[b0 + q] == sv && pt[b0 + q] > tv))) {
          ps[b0 + q + 1] = ps[b0 + q];
          pt[b0 + q + 1] = pt[b0 + q];
          --q;
        }
        ps[b0 + q + 1] = sv;
        pt[b0 + q + 1] = tv;
      }
  }
  __syncthreads();
  const Pool pool{ps, pp, pt};
  const int NL = nfz + nact;  // == w lists
  VS_PROF(true, 2);
  // ---- rank-0 entry = best list head (warp 0) -> δ cutoff ------------------------
  if (wid == 0) {
    int best = -1;
    for (int Lh = lane; Lh < NL; Lh += 32) {
      const int e = Lh < nfz ? Lh : nfz + (Lh - nfz) * Meff;
      if (best < 0 || pool.before(e, best)) best = e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int other = __shfl_xor_sync(FULLM, best, o);
      if (other >= 0 && (best < 0 || pool.before(other, best))) best = other;
    }
    if (lane == 0) s_cut = (cfg.delta != INFINITY && best >= 0) ? ps[best] - cfg.delta : -INFINITY;
  }
  __syncthreads();
  const double cutoff = s_cut;
  // ---- ranks of entries at/above the cutoff --------------------------------------
  const int kk = P < k ? P : k;
  int nkept;
  if (P > 160 && P <= 512) {
    // wide pools: a bitonic sort of the pool indices in proposal order (a
    // strict total order, so the result is the same as ranking each entry);
    // entries at/above the cutoff are a prefix of it (the order is score-first)
    __shared__ short sidx[512];
    int Pp = 256;
    while (Pp < P) Pp <<= 1;
    for (int i = tid; i < Pp; i += NT2) sidx[i] = i < P ? (short)i : (short)-1;
    __syncthreads();
    for (int kb = 2; kb <= Pp; kb <<= 1)
      for (int j = kb >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < Pp; i += NT2) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const int a = sidx[i], c = sidx[ixj];
            const bool a_first = c < 0 || (a >= 0 && pool.before(a, c));
            if (((i & kb) == 0) != a_first) {
              sidx[i] = (short)c;
              sidx[ixj] = (short)a;
            }
          }
        }
        __syncthreads();
      }
    const int e = tid < kk ? sidx[tid] : -1;  // kk <= k <= NT2: one rank per thread
    const bool in = e >= 0 && ps[e] >= cutoff;
    if (in) kept[tid] = e;
    nkept = __syncthreads_count(in);
  } else {
    int mine = 0;
    for (int e = tid; e < P; e += NT2) {
      if (!(ps[e] >= cutoff)) continue;  // pruned by the absolute threshold (inclusive)
      int rank = 0;
      for (int Lh = 0; Lh < NL && rank < kk; ++Lh) {
        const int b0 = Lh < nfz ? Lh : nfz + (Lh - nfz) * Meff;
        const int len = Lh < nfz ? 1 : Meff;
        for (int q = 0; q < len && pool.before(b0 + q, e); ++q) ++rank;  // list is sorted
      }
      if (rank < kk) {
        kept[rank] = e;
        ++mine;
      }
    }
    if (mine) atomicAdd(&s_kept, mine);
    __syncthreads();
    nkept = s_kept;  // ranks 0..nkept-1 are filled (contiguous prefix)
  }

  VS_PROF(true, 3);
  // ---- materialise children (thread j = child j) --------------------------------
  const int j = tid;
  const bool child = j < nkept;
  int pi = 0, tk = -1, clen = 0, crow = 0, src = -1, cfin = 0;
  double csc = 0.0;
  uint64_t chh = 0;
  if (child) {
    const int e = kept[j];
    pi = pp[e];
    tk = pt[e];
    csc = ps[e];
    if (tk < 0) {  // no-op: the finalized candidate itself (bb/search.py:114-115)
      chh = ch[pi];
      clen = cl[pi];
      cfin = 1;
      crow = cr[pi];
      claimed[crow] = 1;
    } else {
      chh = prefix_step(ch[pi], tk);
      clen = cl[pi] + 1;
      cfin = (tk == cfg.eos) || (cl[pi] + 1 >= cfg.max_len);  // bb/core.py:174
      atomicMin(&firstc[pi], j);
    }
  }
  __syncthreads();
  bool extra = false;
  if (child && tk >= 0) {
    if (firstc[pi] == j) {  // the parent's first child inherits its row
      crow = cr[pi];
      claimed[crow] = 1;
    } else {
      extra = true;
      src = cr[pi];
    }
  }
  __syncthreads();
  {
    int nfree, nextra;
    const bool fr = tid < k && !claimed[tid];
    const int fpos = block_prefix(fr, wsm, &nfree);
    if (fr) freel[fpos] = tid;
    const int xpos = block_prefix(extra, wsm, &nextra);  // barrier inside orders freel
    if (extra) {
      crow = freel[xpos];
      act[xpos] = j;  // the pool is built: act[] now lists the extra children
    }
    if (tid == 0) s_nextra = nextra;
  }
  if (child) {
    nrow[j] = crow;
    csrc[j] = src;
    nlen[j] = clen;
    ctok[j] = tk;
    prow[j] = cr[pi];  // a no-op's own row, else the parent's (prefix [0, L))
  }
  VS_PROF(true, 4);
  // ---- deferred emission + length-cap drain ------------------------------------
  const int emitted0 = st.slot_emitted[s];
  int first, ne, width;
  {
    const unsigned bnf = __ballot_sync(FULLM, child && !cfin);
    if (lane == 0) wsm[wid] = bnf ? wid * 32 + __ffs(bnf) - 1 : 0x7fffffff;
    __syncthreads();
    int nlead = nkept;  // leading finalized children
    for (int q = 0; q < NT2 / 32; ++q) nlead = min(nlead, wsm[q]);
    __syncthreads();
    first = min(nlead, k - emitted0);  // pops, bb/search.py:139-141
    ne = first;
    if (child && j < first) emo[j] = j;
    width = nkept - first;
    if (!cfg.no_drain && L + 1 >= cfg.max_len && width > 0) {  // bb/search.py:227-229, :190-202
      const bool rem = child && j >= first;
      int nf_rem, nn_rem;
      const int fpos = block_prefix(rem && cfin, wsm, &nf_rem);
      const int npos = block_prefix(rem && !cfin, wsm, &nn_rem);
      const int quota = k - emitted0 - first;
      if (rem) {
        const int pos = cfin ? fpos : nf_rem + npos;  // finalized first, then capped
        if (pos < quota) emo[first + pos] = j;
      }
      ne = first + min(quota, nf_rem + nn_rem);
      width = 0;
    }
  }
  __syncthreads();
  // emissions append their tokens to out_tok: one atomic per beam reserves them
  {
    int etot;
    const int epre = block_prefix_sum(j < ne ? nlen[emo[j]] : 0, wsm, &etot);
    if (tid == 0 && etot > 0) s_ebase = atomicAdd(&st.counters[6], etot);
    __syncthreads();
    if (j < ne) eoff[j] = s_ebase + epre;
    __syncthreads();
  }
  VS_PROF(true, 5);
  // ---- token histories + emission, one flattened phase ---------------------------
  // Every read is of a claimed row's prefix [0, L) (a parent's, or a no-op's own
  // row), every write goes to a free row or to position L, so the prefix copies
  // of extra children, the appends and the emissions (read from the prefix row
  // + the new token) are independent: no barrier between them, loads batched.
  const int ML = cfg.max_len;
  const int input = st.slot_input[s];
  const int nextra = s_nextra;
  if (child && tk >= 0) st.hist[(int64_t)(base + crow) * ML + L] = tk;
  if (j < ne) {
    const int c = emo[j];
    const int64_t o = (int64_t)input * k + emitted0 + j;
    st.out_len[o] = nlen[c];
    st.out_score[o] = ps[kept[c]];
    st.out_off[o] = eoff[j];
  }
  {
    const int T1 = nextra * L, T = T1 + ne * (L + 1);
    constexpr int U = 4;
    for (int i0 = tid; i0 < T; i0 += NT2 * U) {
      int val[U];
      int32_t* dst[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * NT2;
        dst[u] = nullptr;
        if (i < T1) {  // prefix copy of extra child act[x]
          const int x = i / L, p = i - x * L, c = act[x];
          val[u] = st.hist[(int64_t)(base + csrc[c]) * ML + p];
          dst[u] = st.hist + (int64_t)(base + nrow[c]) * ML + p;
        } else if (i < T) {  // token p of emission q
          const int q = (i - T1) / (L + 1), p = (i - T1) - q * (L + 1), c = emo[q];
          if (p < nlen[c]) {
            const bool last = ctok[c] >= 0 && p == nlen[c] - 1;
            val[u] = last ? ctok[c] : st.hist[(int64_t)(base + prow[c]) * ML + p];
            dst[u] = st.out_tok + (int64_t)eoff[q] + p;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (dst[u]) *dst[u] = val[u];
    }
  }

  VS_PROF(true, 6);
  // ---- next beam SoA, KV copy plan, slot state ---------------------------------
  const bool stays = child && j >= first && j < first + width;
  if (stays) {
    const int d = j - first;
    st.c_score[base + d] = csc;
    st.c_hash[base + d] = chh;
    st.c_len[base + d] = clen;
    st.c_row[base + d] = crow;
    st.c_fin[base + d] = (uint8_t)cfin;
    if (src >= 0 && !cfin) {  // only active children are scored again
      const int slot = atomicAdd(&st.counters[4], 1);  // published as *n_copy by the last CTA
      st.copy_list[3 * slot + 0] = base + src;
      st.copy_list[3 * slot + 1] = base + crow;
      st.copy_list[3 * slot + 2] = L;
    }
  }
  int nact2;  // compact active list of the next beam, in beam order (row list source)
  const int apos = block_prefix(stays && !cfin, wsm, &nact2);
  if (stays && !cfin) st.c_act[base + apos] = act_pack(j - first, crow);
  if (tid == 0) {
    const int emitted = emitted0 + ne;
    st.slot_width[s] = width;
    st.slot_active[s] = nact2;
    st.slot_lt[s] = L + 1;
    st.slot_emitted[s] = emitted;
    st.out_count[input] = emitted;
    const bool finished = width == 0 || emitted >= k || L + 1 >= cfg.max_len;
    if (finished) st.slot_flags[s] |= 2;
  }
}


// ---------------------------------------------------------------------------
// Immediate finalisation policy (bb/search.py:148-187 _expand_immediate):
// the full pool (no M cap) ranked by fp64 SUM; the top-2k scan sends EOS
// proposals straight to the outputs (quota k - emitted) and the rest fill the
// next beam (<= k), δ-pruned against max(first emitted, first fill).  K1
// supplies each parent's top-(2k+2) by (logp desc, token asc): the first 2k+1
// re-sorted by (sum desc, token asc) give the parent's exact top-2k by sum,
// and entry 2k+2 (the best excluded element) is a sentinel proving that no
// excluded element can tie the 2k-th sum through fp64 merging of distinct
// logps (flags InvariantViolation otherwise; needs |score| ~ 2^29 |dlogp|).
__device__ __forceinline__ void beam_immediate(const vs_config& cfg, const vs_state& st, int M_rows,
                                               unsigned char* smem) {
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int k = cfg.k;
  const int s = st.sel[b];
  const int L = st.slot_lt[s];
  const int w = st.slot_width[s];
  const int row0 = st.sel_off[b];
  const int base = s * k;
  const int V = cfg.vocab_size;
  const int Mi = min(2 * k + 1, V);  // list entries per parent (K1 order, re-sorted by sum)
  const int Mu = min(2 * k, V);      // entries a parent can contribute to the scan
  const bool has_sent = V > 2 * k + 1;  // K1 entry 2k+1 = best excluded element
  const int Pmax = k * Mi;

  double* cs = reinterpret_cast<double*>(smem);       // [k]
  uint64_t* ch = reinterpret_cast<uint64_t*>(cs + k);  // [k]
  double* ps = reinterpret_cast<double*>(ch + k);     // [Pmax] sum
  float* pl = reinterpret_cast<float*>(ps + Pmax);    // [Pmax] logp
  int* pp = reinterpret_cast<int*>(pl + Pmax);        // [Pmax] parent
  int* pt = pp + Pmax;                                // [Pmax] token
  int* cl = pt + Pmax;                                // [k]
  int* cr = cl + k;                                   // [k]
  int* scan = cr + k;                                 // [2k] pool index by rank
  int* firstc = scan + 2 * k;                         // [k]
  int* claimed = firstc + k;                          // [k]
  int* freel = claimed + k;                           // [k]
  int* nrow = freel + k;                              // [2k] child row (fill children)
  int* csrc = nrow + 2 * k;                           // [2k]
  __shared__ int wsm[NT2 / 32];
  __shared__ int s_err;

  if (tid < w) {
    cs[tid] = st.c_score[base + tid];
    ch[tid] = st.c_hash[base + tid];
    cl[tid] = st.c_len[base + tid];
    cr[tid] = st.c_row[base + tid];
  }
  if (tid < k) {
    firstc[tid] = 0x7fffffff;
    claimed[tid] = 0;
  }
  if (tid == 0) s_err = 0;
  // bb/search.py:155-158: no finalized candidate may sit on an immediate beam
  if (__syncthreads_or(tid < w && st.c_fin[base + tid] != 0)) {
    if (tid == 0) st.counters[3] = VS_ERR_INVARIANT;
    return;
  }
  // ---- per parent: its Mi entries, re-sorted by (sum desc, token asc) -----------
  for (int a = tid; a < w; a += NT2) {
    const int b0 = a * Mi;
    const double sc = cs[a];
    bool sorted = true;
    for (int m = 0; m < Mi; ++m) {
      const int64_t ri = (int64_t)(row0 + a) * M_rows + m;
      const double lp = row_logp(st, ri);
      pl[b0 + m] = (float)lp;
      pt[b0 + m] = st.top_tok[ri];
      pp[b0 + m] = a;
      ps[b0 + m] = sc + (double)lp;  // bb/search.py:163
      if (m && (ps[b0 + m - 1] < ps[b0 + m] || (ps[b0 + m - 1] == ps[b0 + m] && pt[b0 + m - 1] > pt[b0 + m])))
        sorted = false;
    }
    if (!sorted)
      for (int m = 1; m < Mi; ++m) {
        const double sv = ps[b0 + m];
        const float lv = pl[b0 + m];
        const int tv = pt[b0 + m];
        int q = m - 1;
        while (q >= 0 && (ps[b0 + q] < sv || (ps[b0 + q] == sv && pt[b0 + q] > tv))) {
          ps[b0 + q + 1] = ps[b0 + q];
          pl[b0 + q + 1] = pl[b0 + q];
          pt[b0 + q + 1] = pt[b0 + q];
          --q;
        }
        ps[b0 + q + 1] = sv;
        pl[b0 + q + 1] = lv;
        pt[b0 + q + 1] = tv;
      }
    if (has_sent) {  // boundary proof against the best excluded element
      const int64_t rb = (int64_t)(row0 + a) * M_rows;
      const double lsent = row_logp(st, rb + Mi);
      const int tsent = st.top_tok[rb + Mi];
      const double ssent = sc + lsent;
      const int bT = b0 + Mu - 1;  // the parent's 2k-th entry by sum
      if (ssent == ps[bT] && lsent != -INFINITY) {
        // the sentinel ties the 2k-th sum: it (and the excluded elements tied
        // with it, which have larger tokens) must sort after it, and no excluded
        // element with a smaller logp may round onto the same fp64 sum.  fp64
        // addition is monotone, so the first listed logp below the sentinel's
        // (K1 returns a few slack entries past it) bounds all of them.
        bool bad = tsent < pt[bT];
        if (!bad) {
          int q = Mi + 1;
          while (q < M_rows && row_logp(st, rb + q) == lsent) ++q;
          if (q < M_rows) bad = sc + row_logp(st, rb + q) == ssent;
          else bad = M_rows < V;  // all slack entries tie the sentinel and more exist
        }
        if (bad) s_err = 1;
      }
    }
  }
  __syncthreads();
  if (s_err) {
    if (tid == 0) st.counters[3] = VS_ERR_INVARIANT;
    return;
  }
  // ---- top-2k scan of the pool (parents' first Mu entries) ------------------------
  const Pool pool{ps, pp, pt};
  const int P = w * Mu;
  const int kk = min(2 * k, P);
  for (int e0 = tid; e0 < P; e0 += NT2) {
    const int a = e0 / Mu, m = e0 - a * Mu;
    const int e = a * Mi + m;
    int rank = 0;
    for (int pa = 0; pa < w && rank < kk; ++pa)
      for (int q = 0; q < Mu && pool.before(pa * Mi + q, e); ++q) ++rank;
    if (rank < kk) scan[rank] = e;
  }
  __syncthreads();
  // ---- classify: EOS -> emitted (quota), others -> fill (<= k) ----------------------
  const int emitted0 = st.slot_emitted[s];
  const int quota = k - emitted0;
  const int j = tid;
  const bool in_scan = j < kk;
  const int ej = in_scan ? scan[j] : 0;
  const bool iseos = in_scan && pt[ej] == cfg.eos;
  int n_eos, n_non;
  const int erank = block_prefix(iseos, wsm, &n_eos);
  const int frank = block_prefix(in_scan && !iseos, wsm, &n_non);
  const bool emit = iseos && erank < quota;
  const bool fill = in_scan && !iseos && frank < k;
  const int n_emit = min(n_eos, quota), n_fill = min(n_non, k);
  // anchor = max(first emitted, first fill) (bb/search.py:178-183)
  double anchor = -INFINITY;
  {
    // find first emitted and first fill (lowest scan index of each class)
    const unsigned be = __ballot_sync(FULLM, emit), bf = __ballot_sync(FULLM, fill);
    if (lane == 0) wsm[wid] = (be ? (wid * 32 + __ffs(be) - 1) : 0x7fffffff);
    __syncthreads();
    int fe = 0x7fffffff;
    for (int q = 0; q < NT2 / 32; ++q) fe = min(fe, wsm[q]);
    __syncthreads();
    if (lane == 0) wsm[wid] = (bf ? (wid * 32 + __ffs(bf) - 1) : 0x7fffffff);
    __syncthreads();
    int ff = 0x7fffffff;
    for (int q = 0; q < NT2 / 32; ++q) ff = min(ff, wsm[q]);
    __syncthreads();
    if (fe != 0x7fffffff) anchor = ps[scan[fe]];
    if (ff != 0x7fffffff) anchor = fmax(anchor, ps[scan[ff]]);
  }
  const double cut = cfg.delta != INFINITY ? anchor - cfg.delta : -INFINITY;
  const bool kept = fill && ps[ej] >= cut;  // fill is score-descending: a prefix
  int nkept;
  const int krank = block_prefix(kept, wsm, &nkept);  // child index among kept
  // ---- fill children: rows (first child inherits), tokens, finalisation -------------
  int pi = 0, tk = -1, crow = 0, src = -1, cfin = 0, clen = 0;
  double csc = 0.0;
  uint64_t chh = 0;
  if (kept) {
    pi = pp[ej];
    tk = pt[ej];
    csc = ps[ej];
    chh = prefix_step(ch[pi], tk);
    clen = cl[pi] + 1;
    cfin = clen >= cfg.max_len;  // cannot be EOS here (bb/core.py:174)
    atomicMin(&firstc[pi], krank);
  }
  __syncthreads();
  bool extra = false;
  if (kept) {
    if (firstc[pi] == krank) {
      crow = cr[pi];
      claimed[crow] = 1;
    } else {
      extra = true;
      src = cr[pi];
    }
  }
  __syncthreads();
  {
    int nfree, nextra;
    const bool fr = tid < k && !claimed[tid];
    const int fpos = block_prefix(fr, wsm, &nfree);
    if (fr) freel[fpos] = tid;
    const int xpos = block_prefix(extra, wsm, &nextra);
    if (extra) crow = freel[xpos];
  }
  if (kept) {
    nrow[krank] = crow;
    csrc[krank] = src;
  }
  __syncthreads();
  const int ML = cfg.max_len;
  // every emission of this step (EOS proposals, then the length-cap drain) has
  // L + 1 tokens: one atomic reserves them all in the out_tok append buffer
  const bool drain = !cfg.no_drain && L + 1 >= cfg.max_len && nkept > 0;
  const int nd = drain ? min(k - emitted0 - n_emit, nkept) : 0;
  __shared__ int s_ebase;
  if (tid == 0 && n_emit + nd > 0) s_ebase = atomicAdd(&st.counters[6], (n_emit + nd) * (L + 1));
  __syncthreads();
  const int ebase = s_ebase;
  // ---- EOS emissions straight from the parent's row + eos (warp per emission) -------
  const int input = st.slot_input[s];
  for (int q = wid; q < kk; q += NT2 / 32) {
    const int e = scan[q];
    if (pt[e] != cfg.eos) continue;
    // emission order = scan order among EOS proposals
    int er = 0;
    for (int q2 = 0; q2 < q; ++q2) er += pt[scan[q2]] == cfg.eos;
    if (er >= quota) continue;
    const int64_t o = (int64_t)input * k + emitted0 + er;
    const int64_t to = (int64_t)ebase + (int64_t)er * (L + 1);
    const int32_t* srcp = st.hist + (int64_t)(base + cr[pp[e]]) * ML;
    for (int p = lane; p < L; p += 32) st.out_tok[to + p] = srcp[p];
    if (lane == 0) {
      st.out_tok[to + L] = cfg.eos;
      st.out_len[o] = L + 1;
      st.out_score[o] = ps[e];
      st.out_off[o] = (int32_t)to;
    }
  }
  __syncthreads();  // parents' rows are read above before free rows are overwritten
  for (int c = wid; c < nkept; c += NT2 / 32) {  // prefix copies for extra children
    const int sr = csrc[c];
    if (sr < 0) continue;
    const int32_t* srcp = st.hist + (int64_t)(base + sr) * ML;
    int32_t* dstp = st.hist + (int64_t)(base + nrow[c]) * ML;
    for (int p = lane; p < L; p += 32) dstp[p] = srcp[p];
  }
  __syncthreads();
  if (kept) st.hist[(int64_t)(base + crow) * ML + L] = tk;
  __syncthreads();
  // ---- length-cap drain of the kept fill (all cap-finalised) --------------------------
  int width = nkept, ne = n_emit;
  if (drain) {
    for (int c = wid; c < nd; c += NT2 / 32) {
      const int64_t o = (int64_t)input * k + emitted0 + n_emit + c;
      const int64_t to = (int64_t)ebase + (int64_t)(n_emit + c) * (L + 1);
      const int32_t* srcp = st.hist + (int64_t)(base + nrow[c]) * ML;
      for (int p = lane; p <= L; p += 32) st.out_tok[to + p] = srcp[p];
      if (lane == 0) {
        st.out_len[o] = L + 1;
        st.out_off[o] = (int32_t)to;
      }
    }
    // scores of drained children
    if (kept && krank < nd) st.out_score[(int64_t)input * k + emitted0 + n_emit + krank] = csc;
    ne = n_emit + nd;
    width = 0;
  }
  // ---- next beam SoA, KV copy plan, slot state ---------------------------------
  const bool stays = kept && width > 0;
  if (stays) {
    st.c_score[base + krank] = csc;
    st.c_hash[base + krank] = chh;
    st.c_len[base + krank] = clen;
    st.c_row[base + krank] = crow;
    st.c_fin[base + krank] = (uint8_t)cfin;
    if (src >= 0 && !cfin) {
      const int slot = atomicAdd(&st.counters[4], 1);  // published as *n_copy by the last CTA
      st.copy_list[3 * slot + 0] = base + src;
      st.copy_list[3 * slot + 1] = base + crow;
      st.copy_list[3 * slot + 2] = L;
    }
  }
  int nact2;  // compact active list of the next beam, in beam order (row list source)
  const int apos = block_prefix(stays && !cfin, wsm, &nact2);
  if (stays && !cfin) st.c_act[base + apos] = act_pack(krank, crow);
  if (tid == 0) {
    const int emitted = emitted0 + ne;
    st.slot_width[s] = width;
    st.slot_active[s] = nact2;
    st.slot_lt[s] = L + 1;
    st.slot_emitted[s] = emitted;
    st.out_count[input] = emitted;
    const bool finished = width == 0 || emitted >= k || L + 1 >= cfg.max_len;
    if (finished) st.slot_flags[s] |= 2;
  }
}

// One CTA per slot (grid = n; CTAs past the selection only count in).  The last
// CTA to finish publishes the step's copy count (*n_copy) and, with `sched`,
// runs the scheduler for the next step (removal, refill, selection, row list),
// so K2 and K3 are one launch.
template <bool IMM>
__global__ void __launch_bounds__(NT2) beam_step_kernel(vs_config cfg, vs_state st, int M_rows, int sched, int N,
                                                        int admit_mode, int select_mode, int32_t* mirror) {
  // deferred policy: the PDL wait is inside beam_deferred, after the loads of
  // state the preceding (top-M) kernel does not write; the selected-beam count
  // comes from the previous step's scheduler
  const bool sel = (int)blockIdx.x < __ldcg(&st.status[VS_ST_NSEL]);
  if (IMM || !sel) VS_PDL_ENTRY();
  VS_PROF_T0(true);
  extern __shared__ __align__(16) unsigned char smem[];
  if (sel) {
    if (IMM) beam_immediate(cfg, st, M_rows, smem);
    else beam_deferred(cfg, st, M_rows, smem);
  }
  __syncthreads();
  VS_PROF(true, 7);
  VS_PROF_MAX_FOLD();
  // Grid completion: every other CTA signals its arrival; CTA 0 (always the
  // same CTA, so the scheduler's code stays warm in one SM's instruction
  // cache from step to step) waits for them, publishes the step's copy count
  // and runs the scheduler.  No deadlock: CTA 0 only waits after its own work
  // and occupies one slot while the others run on the remaining ones.
  if (blockIdx.x != 0) {
    if (threadIdx.x == 0) {
      __threadfence();  // this CTA's state writes before its arrival
      atomicAdd(&st.counters[5], 1);
    }
    return;
  }
  if (threadIdx.x == 0) {
    const int want = (int)gridDim.x - 1;
    while (true) {
      int got;
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(got) : "l"(&st.counters[5]) : "memory");
      if (got >= want) break;
      __nanosleep(32);
    }
    st.counters[5] = 0;
    *st.n_copy = atomicExch(&st.counters[4], 0);
    __threadfence();
  }
  __syncthreads();
  VS_PROF(true, 8);
  VS_PROF_MAX_COLLECT();
  if (sched)
    schedule_block<NT2>(cfg, st, N, 0, 1, admit_mode, select_mode, mirror, reinterpret_cast<int*>(smem));
  VS_PROF(true, 15);
  VS_PROF_FLUSH(true);
}

}  // namespace
int32_t* mapped_ptr(void* host);
}  // namespace vs

static int launch_beam_step(const vs_config* cfg, const vs_state* st, int32_t M_rows, int sched, int32_t N,
                            int32_t admit_mode, int32_t select_mode, int32_t* status_mirror, void* stream);

extern "C" int vs_beam_step(const vs_config* cfg, const vs_state* st, int32_t M_rows, void* stream) {
  return launch_beam_step(cfg, st, M_rows, 0, 0, VS_ADMIT_NONE, VS_SELECT_MIN_LT, nullptr, stream);
}

extern "C" int vs_beam_step_schedule(const vs_config* cfg, const vs_state* st, int32_t M_rows, int32_t N,
                                     int32_t admit_mode, int32_t select_mode, int32_t* status_mirror,
                                     void* stream) {
  if (!cfg || cfg->n < 1 || cfg->n > VS_MAX_SLOTS || N < 1 || cfg->capacity < cfg->k) return VS_ERR_CONFIG;
  return launch_beam_step(cfg, st, M_rows, 1, N, admit_mode, select_mode, status_mirror, stream);
}

static int launch_beam_step(const vs_config* cfg, const vs_state* st, int32_t M_rows, int sched, int32_t N,
                            int32_t admit_mode, int32_t select_mode, int32_t* status_mirror, void* stream) {
  if (!cfg || !st || cfg->k < 1 || cfg->k > VS_MAX_K || cfg->max_candidates < 1 ||
      cfg->max_candidates > cfg->k || M_rows < 1)
    return VS_ERR_CONFIG;
  const int k = cfg->k;
  cudaStream_t strm = static_cast<cudaStream_t>(stream);
  int32_t* mirror = vs::mapped_ptr(status_mirror);
  if (status_mirror && !mirror) return VS_ERR_CONFIG;
  const bool imm = cfg->policy == VS_POLICY_IMMEDIATE;
  size_t smem;
  if (imm) {
    const int Mi = min(2 * k + 1, cfg->vocab_size);
    if (M_rows < min(2 * k + 2, cfg->vocab_size) || 2 * k > vs::NT2) return VS_ERR_CONFIG;
    const int Pmax = k * Mi;
    smem = (size_t)2 * k * 8 + (size_t)Pmax * (8 + 4 + 4 + 4) + (size_t)14 * k * 4 + 64;
  } else {
    if (cfg->policy != VS_POLICY_DEFERRED) return VS_ERR_CONFIG;
    const int Meff = cfg->max_candidates < cfg->vocab_size ? cfg->max_candidates : cfg->vocab_size;
    if (M_rows < Meff) return VS_ERR_CONFIG;
    const int Pmax = k + k * Meff;
    smem = (size_t)(2 * k + Pmax) * 8 + (size_t)2 * Pmax * 4 + (size_t)16 * k * 4 + 64;
  }
  if (sched) smem = std::max(smem, vs::sched_smem_bytes(cfg->n));
  if (smem > 200 * 1024) return VS_ERR_CONFIG;
  auto kern = imm ? vs::beam_step_kernel<true> : vs::beam_step_kernel<false>;
  static size_t configured[2] = {0, 0};
  if (smem > 48 * 1024 && smem > configured[imm]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return VS_ERR_CUDA;
    configured[imm] = smem;
  }
  vs::vs_launch(kern, dim3(cfg->n), dim3(vs::NT2), smem, strm, *cfg, *st, M_rows, sched, N, admit_mode,
                select_mode, mirror);
  VS_CUDA_RET();
}

#ifdef VS_PHASE_PROF
// Profiling builds: copy (and reset) the phase accumulators of the fused kernel.
extern "C" int vs_debug_phase_times(unsigned long long* host32) {
  cudaMemcpyFromSymbol(host32, g_prof_acc, 32 * sizeof(unsigned long long));
  static unsigned long long zero[32] = {};
  cudaMemcpyToSymbol(g_prof_acc, zero, sizeof(zero));
  return 0;
}
#endif
