/*
 * varstream.h — C-ABI of the B200-native VarStream search step (sm_100a).
 *
 * The reference (beambatch, pure Python) has no native interface; its plug-in
 * boundary for this path is the per-timestep body of
 *   _execute_step   bb/scheduler.py:168-205  (loop at :180-182)
 * which calls, per selected beam, advance_beam (bb/search.py:215-230) ->
 * expand_beam (bb/search.py:76-103) -> _candidate_pool (:52-73) ->
 * apply_heuristics (bb/heuristics.py:81-93), and, between steps, the
 * ε-refill / min-l_t scheduler (bb/scheduler.py:94-144, :237-287).
 * Each entry point below names the reference function(s) it replaces.
 *
 * Conventions
 *  - Every pointer inside vs_state and every array argument is a DEVICE
 *    pointer allocated by the caller (the library never allocates; all calls
 *    are CUDA-graph capturable).  vs_config / vs_state themselves are host
 *    structs passed by pointer and copied into kernel parameters.
 *  - All calls are asynchronous on `stream` (a cudaStream_t, passed as void*)
 *    and never synchronise the host.
 *  - Return value: VS_OK (0) or a negative VS_ERR_* code for argument errors
 *    detected on the host; device-detected contract breaks are reported in
 *    status[VS_ST_ERROR] (see below).  The Python layer maps them onto the
 *    reference taxonomy (bb/errors.py:10-19): VS_ERR_CONFIG -> ConfigError,
 *    VS_ERR_INVARIANT -> InvariantViolation, VS_ERR_CUDA -> RuntimeError.
 *  - Determinism: every decision is a pure function of the inputs; no
 *    decision depends on atomic ordering.
 */
#ifndef VARSTREAM_H_
#define VARSTREAM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VS_OK 0
#define VS_ERR_CONFIG -1     /* bb/errors.py:13  ConfigError        */
#define VS_ERR_INVARIANT -3  /* bb/errors.py:18  InvariantViolation */
#define VS_ERR_CUDA -4       /* CUDA launch/runtime failure -> RuntimeError */

#define VS_DTYPE_F32 0
#define VS_DTYPE_BF16 1
#define VS_DTYPE_F64 2 /* normalised fp64 log-prob rows only (vs_row_topm_f64) */
/* OR-ed into dtype: rows are already log-probs (reference Scorer rows,
 * bb/model.py:86); lse is taken as 0 so logp = fp32(row). */
#define VS_ROWS_NORMALIZED 0x100
/* OR-ed into dtype for vs_row_lse_topm_ws: pin the K1 kernel (default: the
 * split-row TMA kernel for 8 < M <= 32, the warp-per-row kernel otherwise). */
#define VS_K1_SPLIT 0x200
#define VS_K1_WARP 0x400

#define VS_POLICY_DEFERRED 0  /* bb/core.py:18-28 FinalizationPolicy */
#define VS_POLICY_IMMEDIATE 1

#define VS_ADMIT_NONE -1      /* flush phase: never admit            */
#define VS_ADMIT_VARSTREAM 0  /* live <= floor(eps*n+1e-9)  bb/scheduler.py:335 */
#define VS_ADMIT_VARBEAM 1    /* live == 0                  bb/scheduler.py:306 */
#define VS_ADMIT_VARFIFO 2    /* live <  n                  bb/scheduler.py:359 */

#define VS_SELECT_MIN_LT 0    /* bb/scheduler.py:135-144 */
#define VS_SELECT_FIFO 1      /* bb/scheduler.py:147-157 */
#define VS_SELECT_ALL 2       /* bb/scheduler.py:160-165 (flush) */

/* Limits of this build. */
#define VS_MAX_K 128
#define VS_MAX_M 128
#define VS_MAX_SLOTS 1024

/* Search/scheduling knobs: the resolved bb/core.py:88-140 DecodeConfig. */
typedef struct vs_config {
  int32_t k;                /* beam width                                   */
  int32_t n;                /* batch size (number of beam slots)            */
  int32_t max_candidates;   /* M, per-parent cap                            */
  int32_t max_len;          /* length cap (tokens incl. sos)                */
  int32_t vocab_size;       /* |V|                                          */
  int32_t sos, eos;
  int32_t policy;           /* VS_POLICY_*                                  */
  int32_t capacity;         /* max rows scored per step                     */
  int32_t refill_threshold; /* floor(eps*n + 1e-9)  bb/scheduler.py:237-240 */
  int32_t no_drain;         /* 1: expand only (bb/search.py:76 expand_beam),
                               0: advance (adds the length-cap drain :227-229) */
  double delta;             /* absolute threshold; +inf disables            */
} vs_config;

/* Status record written by vs_schedule (int32 slots, host reads it each step). */
#define VS_ST_R 0           /* rows to score this step (expansions)         */
#define VS_ST_NSEL 1        /* number of selected beams                     */
#define VS_ST_NLIVE 2       /* live beams after refill                      */
#define VS_ST_L 3           /* effective_len of the selection               */
#define VS_ST_NADMIT 4      /* inputs admitted at the top of this step      */
#define VS_ST_ADMIT0 5      /* first admitted input id (admits are consecutive) */
#define VS_ST_CURSOR 6      /* stream cursor after refill                   */
#define VS_ST_DONE 7        /* 1 when no live beams remain and stream is empty */
#define VS_ST_ERROR 8       /* 0 or VS_ERR_*                                */
#define VS_ST_NFIN 9        /* beams removed as finished (previous step)    */
#define VS_ST_NLIVE_AFTER 10 /* live count right after removal               */
#define VS_ST_TOKFILL 11    /* tokens appended to out_tok so far this run   */
#define VS_ST_MINLIVE 12    /* every input below this id is finished: its
                               outputs (and their tokens, all below
                               TOKFILL) are final                           */
#define VS_ST_HDR 16
/* followed by: selected input ids [n], finished input ids [n],
 * live-after-removal input ids [n], admitted slot ids [n]  (total HDR+4n). */
#define VS_STATUS_INTS(n) (VS_ST_HDR + 4 * (n))

/* Device-resident state of one refilling batch.  Slots never move; the live
 * list is an index list in arrival order (bb/scheduler.py:57-65).  Candidate
 * j of slot s lives at [s*k + j] (score-descending beam order,
 * bb/core.py:64-77); c_row maps it to its PHYSICAL row s*k + c_row, which
 * owns the token history (and any scorer per-row state such as a KV cache). */
typedef struct vs_state {
  /* per slot [n] */
  int32_t* slot_input;   /* input id (corpus position)                  */
  int32_t* slot_lt;      /* l_t                                         */
  int32_t* slot_emitted; /* candidates emitted so far                   */
  int32_t* slot_width;   /* candidates on the beam                      */
  int32_t* slot_active;  /* non-finalized candidates (active width)     */
  int32_t* slot_src_len; /* source length                               */
  int32_t* slot_flags;   /* bit0 used, bit1 finished (set by beam_step) */
  uint64_t* slot_seed;   /* scorer per-source seed (hash scorer)         */
  /* per candidate [n*k] */
  double* c_score;       /* cumulative log-prob, fp64 (bb/core.py:173)  */
  int32_t* c_len;        /* token count                                 */
  int32_t* c_row;        /* physical row within the slot [0,k)          */
  uint8_t* c_fin;        /* finalized                                   */
  uint64_t* c_hash;      /* prefix hash (candidate fingerprint)         */
  /* per physical row [n*k, max_len] */
  int32_t* hist;         /* token history                               */
  /* scheduler */
  int32_t* live;         /* [n] slot ids in arrival order               */
  int32_t* counters;     /* [8]: n_live, cursor, N, error, copy counter,
                            CTA arrival counter, out_tok fill
                            (zero-initialised)                          */
  int32_t* sel;          /* [n] selected slot ids, in advance order     */
  int32_t* sel_off;      /* [n+1] row offsets of selected beams         */
  int32_t* row_slot;     /* [capacity] slot of each scored row          */
  int32_t* row_cand;     /* [capacity] candidate index within the beam  */
  int32_t* row_phys;     /* [capacity] physical row (s*k + c_row)       */
  int32_t* row_len;      /* [capacity] candidate length (= l_t)         */
  /* corpus [N] (device copy of the length-bucketed stream) */
  const int32_t* src_off; /* [N+1] offsets into src_tok                 */
  const int32_t* src_tok; /* flat source tokens                         */
  /* outputs */
  int32_t* out_count;    /* [N]                                         */
  int32_t* out_len;      /* [N*k]                                       */
  double* out_score;     /* [N*k]                                       */
  int32_t* out_tok;      /* append buffer (capacity N*k*max_len): the
                            emitted candidates' tokens back to back     */
  /* per-row top-M (written by the row kernel) [capacity*M] */
  int32_t* top_tok;
  float* top_logp;
  float* row_lse;        /* [capacity]                                  */
  /* KV / row-state copies planned by beam_step: (src_phys, dst_phys, len) */
  int32_t* copy_list;    /* [n*k*3]: <= k surviving children per beam   */
  int32_t* n_copy;       /* [1] copies planned by the last beam step    */
  /* host-visible status (VS_STATUS_INTS(n)) */
  int32_t* status;
  /* per candidate [n*k]: the beam's ACTIVE candidates in beam order, packed
   * (cand | phys_row << 8), written by the beam step and by admission; the
   * scheduler builds the next row list from it */
  int32_t* c_act;
  /* [capacity*M] fp64 row values of the top-M entries, or NULL.  Set when the
   * rows are reference fp64 log-probs (vs_row_topm_f64): the beam step then
   * adds these exact values instead of the fp32 top_logp (bb/search.py:71). */
  double* top_logp64;
  /* [N*k] start of each emitted candidate's tokens in out_tok */
  int32_t* out_off;
} vs_state;

/* Library identification / sanity. */
int vs_version(void);

/* K1  row_lse_topM — replaces bb/model.py:216-217 (log-softmax) and
 * bb/search.py:63-73 (per-parent top-M by (row value desc, token asc)).
 * For each row r < R (R = *d_R when d_R != NULL, else R_host):
 *   lse[r] = max + log(sum exp(x - max))          (fp32)
 *   logp   = fp32(x - lse[r])
 *   top-M tokens by (logp desc, token asc) -> top_tok[r*M+j], top_logp[r*M+j]
 * Rows are read once from HBM (16-byte vector loads) with an exact fallback
 * for rows whose boundary is ambiguous; M <= VS_MAX_M.  If V < M the tail of
 * each output row is filled with token -1 / logp -inf. */
int vs_row_lse_topm(const void* logits, int32_t dtype, int64_t ld, int32_t V, int32_t M,
                    int32_t R_host, const int32_t* d_R, int32_t R_grid, int32_t* top_tok,
                    float* top_logp, float* row_lse, int32_t* fallback_count, void* stream);

/* K1-f64 — per-row top-M over NORMALISED fp64 log-prob rows (the rows a
 * reference Scorer returns, bb/model.py:86, :216-217): top-M tokens by
 * (row value desc, token asc) (bb/search.py:69), the exact fp64 values into
 * top_logp64 (and, if non-NULL, their fp32 roundings into top_logp).  NaN
 * entries never rank; V < M pads with token -1 / -inf.  Parity path for host
 * scorers: one warp per row, M arg-max rounds. */
int vs_row_topm_f64(const double* rows, int64_t ld, int32_t V, int32_t M, int32_t R_host,
                    const int32_t* d_R, int32_t R_grid, int32_t* top_tok, float* top_logp,
                    double* top_logp64, void* stream);

/* K1 with a caller-provided workspace — same contract and outputs as
 * vs_row_lse_topm.  When the rows qualify (16-byte aligned logits and
 * ld*sizeof(T), 4 KB <= V*sizeof(T) <= 256 KB, M <= 32) it runs the
 * TMA-staged split-row kernel (csrc/row_topm_tma.cu): a persistent grid whose
 * warps stream equal slices of the R x |V| logits through cp.async.bulk
 * shared-memory rings, so small steps still fill all 148 SMs.  Its lse is a
 * partition-invariant function of the row (independent of R).  Otherwise it
 * behaves exactly like vs_row_lse_topm.  The workspace must hold
 * vs_row_lse_topm_ws_bytes(R_grid, V, dtype) bytes and be ZEROED ONCE when
 * allocated (per-row counters return to zero after every launch). */
int vs_row_lse_topm_ws(const void* logits, int32_t dtype, int64_t ld, int32_t V, int32_t M,
                       int32_t R_host, const int32_t* d_R, int32_t R_grid, int32_t* top_tok,
                       float* top_logp, float* row_lse, int32_t* fallback_count, void* workspace,
                       size_t workspace_bytes, void* stream);
size_t vs_row_lse_topm_ws_bytes(int32_t R_grid, int32_t V, int32_t dtype);

/* K2  beam_step — replaces bb/search.py:76-145 (expand_beam, deferred),
 * :148-187 (immediate), :190-230 (length-cap drain, advance_beam) and
 * bb/heuristics.py:42-93 (cap + δ threshold), and the per-slot loop body of
 * bb/scheduler.py:180-182 + the finished test :190-192.  One CTA per
 * selected beam; emits finalized candidates into the output buffers and plans
 * row-state copies (copy_list) for the KV reorder (vs_rows_copy).  For the
 * immediate policy the caller passes per-row top-(2k) by (logp desc, token
 * asc) in top_tok/top_logp with M = min(2k, V). */
int vs_beam_step(const vs_config* cfg, const vs_state* st, int32_t M_rows, void* stream);

/* K2+K3 fused — the same beam step, whose LAST CTA to finish then runs the
 * scheduler for the next step (vs_schedule with do_remove=1, first_call=0 and
 * the given modes): one launch per search step after the row kernel.  The
 * status header is also written to status_mirror (16 int32 in pinned host
 * memory, or NULL), so a host-side ring needs no copy launch.  Replaces
 * bb/scheduler.py:180-192 + the next iteration's :266-270. */
int vs_beam_step_schedule(const vs_config* cfg, const vs_state* st, int32_t M_rows, int32_t N,
                          int32_t admit_mode, int32_t select_mode, int32_t* status_mirror, void* stream);

/* K3  compact_refill_select — replaces bb/scheduler.py:190-192 (stable
 * removal of finished beams), :94-116 + :237-240 + :266-268 (ε-refill),
 * :119-165 (min-l_t / FIFO / all selection with capacity packing) and builds
 * the next step's row list.  first_call=1 initialises the counters.
 * admit_mode: VS_ADMIT_*; select_mode: VS_SELECT_*; do_remove: apply the
 * previous step's finished flags first. */
int vs_schedule(const vs_config* cfg, const vs_state* st, int32_t N, int32_t first_call,
                int32_t do_remove, int32_t admit_mode, int32_t select_mode, void* stream);
/* vs_schedule that also writes the status header to status_mirror (pinned
 * host memory, 16 int32). */
int vs_schedule_mirror(const vs_config* cfg, const vs_state* st, int32_t N, int32_t first_call,
                       int32_t do_remove, int32_t admit_mode, int32_t select_mode, int32_t* status_mirror,
                       void* stream);

/* K4  row-state reorder — no reference equivalent (the reference scorer is
 * stateless; bb/core.py:170 copies token tuples).  Applies copy_list: for
 * each (src, dst, len) copies positions [0,len) of `planes` planes, each
 * plane laid out as [rows, pos_stride_bytes*max_pos] with plane_stride_bytes
 * between planes.  pos_bytes < 0 selects fixed-size records: every copy
 * moves exactly -pos_bytes bytes (per-row recurrent state such as an LSTM's
 * (h, c)), whatever its len.  Sources are never destinations (by construction in
 * vs_beam_step), so the copy is hazard-free in place. */
int vs_rows_copy(void* base, int64_t plane_stride_bytes, int32_t planes, int64_t row_stride_bytes,
                 int64_t pos_bytes, const int32_t* copy_list, const int32_t* n_copy,
                 int32_t max_copies, void* stream);

/* Encoder-state placement (K4 second half): scatter `count` rows of `bytes`
 * each from src (dense) into dst at row index slots[i] (row stride dst_stride). */
int vs_scatter_rows(void* dst, int64_t dst_stride_bytes, const void* src, int64_t src_stride_bytes,
                    int64_t bytes, const int32_t* slots, const int32_t* d_count, int32_t count_max,
                    void* stream);

/* Row LayerNorm without affine for bf16 activations (the decoder scorers):
 * y[r] = (x[r] - mean) * rsqrt(var + eps), fp32 statistics, bf16 out; warp per
 * row; d a multiple of 256 up to 4096, 16-byte aligned rows. */
int vs_layer_norm_bf16(const void* x, int64_t ldx, void* y, int64_t ldy, int32_t R, int32_t d, float eps,
                       void* stream);

/* Synthetic device scorer (stands in for the decoder's logits; mirrors the
 * structure of bb/model.py:209-218 SeededHashScorer with an integer hash).
 * vs_hash_encode: per admitted slot (status admitted list) computes the
 * source seed and the initial candidate hash.  vs_hash_logits: writes
 * logits[r, v] for r < R (device R = status[VS_ST_R]). */
typedef struct vs_hash_params {
  uint64_t seed;
  float scale;
  float eos_bias;
  int32_t power; /* 1, 2 or 4 */
  int32_t dtype; /* VS_DTYPE_* */
} vs_hash_params;

int vs_hash_encode(const vs_config* cfg, const vs_state* st, uint64_t seed, void* stream);
int vs_hash_logits(const vs_config* cfg, const vs_state* st, const vs_hash_params* hp,
                   void* logits, int64_t ld, int32_t R_grid, void* stream);

/* Decode attention over physical rows (decoder scorer).
 * For each row r < R (R = *d_R when d_R != NULL, else R_host; grid R_grid):
 *   out[r, h, :] = softmax_t(q[r,h,:] . K[idx[r], t, h, :] * scale) @ V[idx[r], t, h, :]
 * over t < lens[r].  K/V element (row, t, h, e) lives at
 * row*row_stride + t*pos_stride + h*head_dim + e (bf16).  With k_new/v_new
 * (bf16 [R, heads*head_dim], row stride new_ld) position lens[r]-1 is taken from
 * them and written into the cache first (self-attention append).  head_dim must
 * be 64, heads a multiple of 4, lens[r] <= 256.  Replaces nothing in the reference (its
 * scorer is stateless, bb/model.py:78-87); it is the batched scorer's kernel. */
int vs_row_attention(const void* q, int64_t q_ld, void* k_cache, void* v_cache, int64_t row_stride,
                     int64_t pos_stride, const int32_t* idx, const int32_t* lens, const void* k_new,
                     const void* v_new, int64_t new_ld, void* out, int64_t out_ld, int32_t heads,
                     int32_t head_dim, float scale, int32_t R_host, const int32_t* d_R, int32_t R_grid,
                     void* stream);

/* Grouped decode attention (no append) for rows that share one cache row:
 * group g (g < *d_ngroups, G_grid bounds it) is rows [grp_off[g], grp_off[g+1]),
 * all with the same idx and lens (the cross-attention of one beam: grp_off =
 * the engine's sel_off, *d_ngroups = status[VS_ST_NSEL]).  One CTA per
 * (group, head) stages the shared K/V lines (and 64 query rows at a time) in
 * shared memory once and runs mma.m16n8k16 tiles with an online softmax (P in
 * bf16, fp32 accumulation).  head_dim 64, lens <= 256. */
int vs_row_attention_grouped(const void* q, int64_t q_ld, const void* k_cache, const void* v_cache,
                             int64_t row_stride, int64_t pos_stride, const int32_t* idx, const int32_t* lens,
                             const int32_t* grp_off, const int32_t* d_ngroups, int32_t G_grid, void* out,
                             int64_t out_ld, int32_t heads, int32_t head_dim, float scale, void* stream);

/* K5  proj_lse_topM — the decoder's vocab projection on tcgen05 tensor cores
 * with K1 fused into the epilogue (csrc/proj_topm.cu).  For rows r < R
 * (R = *d_R when d_R != NULL, else R_host; R_grid bounds R and sizes the TMA
 * map of H):
 *   x[r, v] = bf16(H[r, :] . W[v, :]), x[r, eos] = bf16(x[r, eos] + eos_add[r])
 *   lse[r], top-M by (logp desc, token asc) — K1's contract on x.
 * H: bf16 [R_grid, K] (row stride ldh), W: bf16 [V, K] (row stride ldw), K a
 * multiple of 64, M <= 8, |V| <= 65536.  logits (bf16 [R, ldo], required)
 * receives x: the merge reads only the few 128-column sub-tiles that can hold
 * a row's top-M, and the exact fallback reads the row.  Workspace:
 * vs_proj_lse_topm_ws_bytes(R_grid, V) bytes (no zeroing needed).  Replaces the vocab GEMM + bb/model.py:216-217 +
 * bb/search.py:63-73. */
int vs_proj_lse_topm(const void* H, int64_t ldh, const void* W, int64_t ldw, int32_t R_host,
                     const int32_t* d_R, int32_t R_grid, int32_t K, int32_t V, int32_t M, int32_t eos,
                     const float* eos_add, void* logits, int64_t ldo, int32_t* top_tok, float* top_logp,
                     float* row_lse, int32_t* fallback_count, void* workspace, size_t workspace_bytes,
                     void* stream);
size_t vs_proj_lse_topm_ws_bytes(int32_t R_grid, int32_t V);

#ifdef __cplusplus
}
#endif
#endif /* VARSTREAM_H_ */
