// K2 beam_step: per-beam merge, δ/M pruning, EOS finalisation, emission,
// length-cap drain and row planning (sm_100a).  One CTA per selected beam.
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
// Row planning (new, no reference equivalent): candidates are logical; each
// owns a physical row of the slot (token history + scorer row state such as
// a KV cache).  The first child of a parent inherits the parent's row (no
// copy); further children take rows freed by parents without surviving
// children and get a (src,dst,len) copy entry.  Sources are always rows
// claimed by inheritors, destinations always free rows, so in-place copies
// are hazard-free.
//
// The per-parent cap never binds here: each parent contributes exactly
// min(M, V) proposals (pre-truncated by K1), so max_candidates_filter accepts
// every extension and the kept set is the first min(k, |pool|) in order.
#include "common.cuh"

namespace vs {
namespace {

struct PoolView {
  const double* sc;
  const int* par;
  const int* tok;
  // true when entry f precedes e in proposal_order (score desc, parent asc, token asc)
  __device__ __forceinline__ bool before(int f, int e) const {
    const double a = sc[f], b = sc[e];
    if (a != b) return a > b;
    if (par[f] != par[e]) return par[f] < par[e];
    return tok[f] < tok[e];
  }
};

constexpr int NT2 = 128;

__global__ void __launch_bounds__(NT2) beam_step_kernel(vs_config cfg, vs_state st, int M_rows) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int b = blockIdx.x;
  if (b >= st.status[VS_ST_NSEL]) return;
  const int tid = threadIdx.x;
  const int k = cfg.k;
  const int s = st.sel[b];
  const int L = st.slot_lt[s];
  const int w = st.slot_width[s];
  const int row0 = st.sel_off[b];
  const int base = s * k;
  const int Meff = cfg.max_candidates < cfg.vocab_size ? cfg.max_candidates : cfg.vocab_size;
  const int Pmax = k + k * Meff;

  // ---- shared memory carve-up -------------------------------------------------
  double* cs = reinterpret_cast<double*>(smem);  // [k]  current scores
  uint64_t* ch = reinterpret_cast<uint64_t*>(cs + k);  // [k]
  double* ps = reinterpret_cast<double*>(ch + k);  // [Pmax] pool score
  double* ns = ps + Pmax;                           // [k] child score
  uint64_t* nh = reinterpret_cast<uint64_t*>(ns + k);  // [k] child hash
  int* pp = reinterpret_cast<int*>(nh + k);         // [Pmax] pool parent
  int* pt = pp + Pmax;                              // [Pmax] pool token (-1 = no-op)
  int* cl = pt + Pmax;                              // [k] current len
  int* cr = cl + k;                                 // [k] current row
  int* act = cr + k;                                // [k] active ordinal -> cand idx
  int* fin = act + k;                               // [k] finalized ordinal -> cand idx
  int* kept = fin + k;                              // [k] pool index by rank
  int* nrow = kept + k;                             // [k] child row
  int* nsrc = nrow + k;                             // [k] copy source row (-1 none)
  int* nlen = nsrc + k;                             // [k] child len
  int* ntok = nlen + k;                             // [k] appended token (-1 none)
  int* nfin = ntok + k;                             // [k] child finalized
  int* emo = nfin + k;                              // [k] emission order -> child idx
  int* claimed = emo + k;                           // [k]
  int* inh = claimed + k;                           // [k]
  __shared__ int wcnt[2][NT2 / 32];
  __shared__ int sh[8];  // 0 nact 1 nfin 2 nkept 3 nemit 4 first_remaining 5 emitted_after 6 next_width

  // candidates -> smem (parallel loads; w <= k <= 128 = NT2)
  for (int i = tid; i < w; i += NT2) {
    cs[i] = st.c_score[base + i];
    ch[i] = st.c_hash[base + i];
    cl[i] = st.c_len[base + i];
    cr[i] = st.c_row[base + i];
  }
  {  // stable split into finalized / active ordinals via warp ballots
    const int lane = tid & 31, wid = tid >> 5;
    const bool valid = tid < w;
    const bool f = valid && st.c_fin[base + tid] != 0;
    const unsigned bf = __ballot_sync(0xffffffffu, f);
    const unsigned ba = __ballot_sync(0xffffffffu, valid && !f);
    if (lane == 0) {
      wcnt[0][wid] = __popc(bf);
      wcnt[1][wid] = __popc(ba);
    }
    __syncthreads();
    int fo = 0, ao = 0;
    for (int q = 0; q < wid; ++q) {
      fo += wcnt[0][q];
      ao += wcnt[1][q];
    }
    const unsigned lt_mask = (1u << lane) - 1u;
    if (f) fin[fo + __popc(bf & lt_mask)] = tid;
    if (valid && !f) act[ao + __popc(ba & lt_mask)] = tid;
    if (tid == 0) {
      int na = 0, nf = 0;
      for (int q = 0; q < NT2 / 32; ++q) {
        nf += wcnt[0][q];
        na += wcnt[1][q];
      }
      sh[0] = na;
      sh[1] = nf;
    }
  }
  __syncthreads();
  const int nact = sh[0], nfz = sh[1];
  const int P = nfz + nact * Meff;

  // ---- pool (bb/search.py:64-72): no-ops then per-parent top-M ------------------
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
      ps[e] = cs[i] + (double)st.top_logp[ri];  // fp64 add, bb/search.py:71
      pp[e] = i;
      pt[e] = st.top_tok[ri];
    }
  }
  __syncthreads();

  // ---- first min(k, P) in proposal_order: exact rank counting with early exit ----
  // Scan order visits no-ops then every parent's best proposals first, so
  // entries outside the top-k stop after ~k comparisons.
  const int kk = P < k ? P : k;
  const PoolView pv{ps, pp, pt};
  for (int e = tid; e < P; e += NT2) {
    int rank = 0;
    for (int j = 0; j < P && rank < kk; ++j) {
      int f;
      if (j < nfz) f = j;
      else {
        const int jj = j - nfz, m = jj / nact, a = jj - m * nact;
        f = nfz + a * Meff + m;
      }
      rank += pv.before(f, e);
    }
    if (rank < kk) kept[rank] = e;
  }
  __syncthreads();

  // ---- threshold, materialisation, row plan, emission, drain (one thread) ------
  if (tid == 0) {
    int nk = kk;
    if (cfg.delta != INFINITY) {  // bb/heuristics.py:75-78, anchor = kept[0]
      const double cutoff = ps[kept[0]] - cfg.delta;
      int j = 0;
      while (j < nk && ps[kept[j]] >= cutoff) ++j;
      nk = j;
    }
    for (int r = 0; r < k; ++r) {
      claimed[r] = 0;
      inh[r] = 0;
    }
    for (int j = 0; j < nk; ++j) {
      const int e = kept[j], i = pp[e], t = pt[e];
      ns[j] = ps[e];
      if (t < 0) {  // no-op: the finalized candidate itself
        nh[j] = ch[i];
        nlen[j] = cl[i];
        ntok[j] = -1;
        nfin[j] = 1;
        nrow[j] = cr[i];
        nsrc[j] = -1;
        claimed[cr[i]] = 1;
      } else {
        nh[j] = prefix_step(ch[i], t);
        nlen[j] = cl[i] + 1;
        ntok[j] = t;
        nfin[j] = (t == cfg.eos) || (cl[i] + 1 >= cfg.max_len);  // bb/core.py:174
        if (!inh[i]) {
          inh[i] = 1;
          nrow[j] = cr[i];
          nsrc[j] = -1;
          claimed[cr[i]] = 1;
        } else {
          nrow[j] = -1;
          nsrc[j] = cr[i];
        }
      }
    }
    int fr = 0;
    for (int j = 0; j < nk; ++j) {
      if (nrow[j] >= 0) continue;
      while (claimed[fr]) ++fr;
      nrow[j] = fr;
      claimed[fr] = 1;
    }
    // deferred emission: pop rank-1 finalized while emitted < k (bb/search.py:139-141)
    int emitted = st.slot_emitted[s];
    int ne = 0, first = 0;
    while (first < nk && nfin[first] && emitted < k) {
      emo[ne++] = first++;
      ++emitted;
    }
    int width = nk - first;
    // length-cap drain (bb/search.py:227-229, :190-202): finalized, then capped
    if (!cfg.no_drain && L + 1 >= cfg.max_len && width > 0) {
      for (int pass = 0; pass < 2; ++pass)
        for (int j = first; j < nk; ++j) {
          if ((pass == 0) != (nfin[j] != 0)) continue;
          if (emitted >= k) break;
          emo[ne++] = j;
          ++emitted;
        }
      width = 0;
      first = nk;
    }
    sh[2] = nk;
    sh[3] = ne;
    sh[4] = first;
    sh[5] = emitted;
    sh[6] = width;
  }
  __syncthreads();
  const int nk = sh[2], ne = sh[3], first = sh[4], width = sh[6];
  const int ML = cfg.max_len;

  // ---- token histories: copy parent prefix into new rows, then append -------
  for (int j = 0; j < nk; ++j) {
    if (nsrc[j] < 0) continue;
    const int32_t* src = st.hist + (int64_t)(base + nsrc[j]) * ML;
    int32_t* dst = st.hist + (int64_t)(base + nrow[j]) * ML;
    for (int p = tid; p < L; p += NT2) dst[p] = src[p];
  }
  __syncthreads();
  for (int j = tid; j < nk; j += NT2)
    if (ntok[j] >= 0) st.hist[(int64_t)(base + nrow[j]) * ML + L] = ntok[j];
  __syncthreads();

  // ---- emission into the per-input output buffers ----------------------------
  const int input = st.slot_input[s];
  const int e0 = st.slot_emitted[s];
  for (int q = 0; q < ne; ++q) {
    const int j = emo[q];
    const int64_t o = (int64_t)input * k + e0 + q;
    const int32_t* src = st.hist + (int64_t)(base + nrow[j]) * ML;
    for (int p = tid; p < nlen[j]; p += NT2) st.out_tok[o * ML + p] = src[p];
    if (tid == 0) {
      st.out_len[o] = nlen[j];
      st.out_score[o] = ns[j];
    }
  }

  // ---- next beam SoA, KV copy plan, slot state ---------------------------------
  for (int j = tid; j < width; j += NT2) {
    const int c = first + j;
    st.c_score[base + j] = ns[c];
    st.c_hash[base + j] = nh[c];
    st.c_len[base + j] = nlen[c];
    st.c_row[base + j] = nrow[c];
    st.c_fin[base + j] = (uint8_t)nfin[c];
    if (nsrc[c] >= 0 && !nfin[c]) {  // only active children are scored again
      const int slot = atomicAdd(st.n_copy, 1);
      st.copy_list[3 * slot + 0] = base + nsrc[c];
      st.copy_list[3 * slot + 1] = base + nrow[c];
      st.copy_list[3 * slot + 2] = L;
    }
  }
  if (tid == 0) {
    int nact2 = 0;
    for (int j = first; j < first + width; ++j) nact2 += !nfin[j];
    const int emitted = sh[5];
    st.slot_width[s] = width;
    st.slot_active[s] = nact2;
    st.slot_lt[s] = L + 1;
    st.slot_emitted[s] = emitted;
    st.out_count[input] = emitted;
    const bool finished = width == 0 || emitted >= k || L + 1 >= cfg.max_len;
    if (finished) st.slot_flags[s] |= 2;
  }
}

}  // namespace
}  // namespace vs

extern "C" int vs_beam_step(const vs_config* cfg, const vs_state* st, int32_t M_rows, void* stream) {
  if (!cfg || !st || cfg->k < 1 || cfg->k > VS_MAX_K || cfg->max_candidates < 1 ||
      cfg->max_candidates > cfg->k || M_rows < 1)
    return VS_ERR_CONFIG;
  if (cfg->policy != VS_POLICY_DEFERRED) return VS_ERR_CONFIG;  // immediate: see DESIGN.md
  const int k = cfg->k;
  const int Meff = cfg->max_candidates < cfg->vocab_size ? cfg->max_candidates : cfg->vocab_size;
  if (M_rows < Meff) return VS_ERR_CONFIG;
  const int Pmax = k + k * Meff;
  const size_t smem = (size_t)(4 * k + Pmax) * 8 /*cs,ch,ns,nh + ps*/ + (size_t)2 * Pmax * 4 +
                      (size_t)15 * k * 4 + 64;
  if (smem > 200 * 1024) return VS_ERR_CONFIG;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    if (cudaFuncSetAttribute(vs::beam_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return VS_ERR_CUDA;
    configured = smem;
  }
  vs::beam_step_kernel<<<cfg->n, vs::NT2, smem, static_cast<cudaStream_t>(stream)>>>(*cfg, *st, M_rows);
  VS_CUDA_RET();
}
