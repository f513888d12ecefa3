// K3 compact_refill_select as a block-level device routine (sm_100a), shared
// by the standalone scheduler launch (csrc/schedule.cu) and the fused
// beam-step kernel, whose LAST CTA to finish runs it (csrc/beam_step.cu), so a
// search step is one launch after the row kernel.
//
//   A. stable removal of finished beams      bb/scheduler.py:190-192 (+ finished
//      ids in selection order :186-189 for StepEvent)
//   B. ε-refill at the top of the step        bb/scheduler.py:94-116, :237-240,
//      admit predicates :306 / :335 / :359, checked once (:266-268)
//   C. selection with capacity packing       bb/scheduler.py:119-165
//      (min-l_t in arrival order / FIFO most-advanced first / all for flush;
//      greedy arrival-order fill, skip and continue; width > capacity ->
//      ConfigError :125-128)
//   D. the next step's row list: active candidates of the selected beams in
//      beam order (bb/search.py:223-225), copied from each slot's compact
//      active list c_act (written by the beam step): one independent load per
//      row, all threads of the block.
//
// A-C touch at most n <= 1024 slots and are latency-bound: every thread owns
// a contiguous run of ceil(n / NT) items and every stable compaction is one
// block scan of per-thread counts (one warp looping over n / 32 items per lane
// measured ~28k cycles on the fused launch's scheduler CTA).  All per-slot state is pulled
// into shared memory in one round of independent loads.  Slots never move:
// the live list is an index list and admission takes the lowest free slot ids
// (placement does not affect results).
#pragma once
#include "common.cuh"

namespace vs {

constexpr unsigned SCHED_FULL = 0xffffffffu;

// Warp exclusive scan of one int per lane; total in *tot.
__device__ __forceinline__ int warp_excl_scan(int v, int* tot) {
  const int lane = threadIdx.x & 31;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(SCHED_FULL, x, o);
    if (lane >= o) x += y;
  }
  *tot = __shfl_sync(SCHED_FULL, x, 31);
  return x - v;
}

__device__ __forceinline__ int warp_min_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(SCHED_FULL, v, o));
  return v;
}

// Block-wide (NT threads) exclusive scan of one int per thread; total in *tot.
// wsum holds NT / 32 ints of shared memory.  Contains two block barriers.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int* tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(SCHED_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  int off = 0, t = 0;
#pragma unroll
  for (int q = 0; q < NT / 32; ++q) {
    const int wq = wsum[q];
    off += q < wid ? wq : 0;
    t += wq;
  }
  __syncthreads();
  *tot = t;
  return off + x - v;
}

template <int NT>
__device__ __forceinline__ int block_min(int v, int* wsum) {
  v = warp_min_i(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) wsum[wid] = v;
  __syncthreads();
  int m = 0x7fffffff;
#pragma unroll
  for (int q = 0; q < NT / 32; ++q) m = min(m, wsum[q]);
  __syncthreads();
  return m;
}

// Shared-memory bytes schedule_block needs for n slots (+ 32 ints of block-scan partials).
__host__ __device__ constexpr size_t sched_smem_bytes(int n) { return (size_t)(9 * n + 1 + 8 + 32) * 4; }

// Packed active-list entry (beam step -> scheduler): candidate index and its
// physical row within the slot (both < VS_MAX_K = 128).
__device__ __forceinline__ int act_pack(int cand, int row) { return cand | (row << 8); }

// The scheduler step, run by all NT threads of a block.  `smem` holds
// sched_smem_bytes(cfg.n) bytes; `mirror` (host-mapped pinned memory, or
// nullptr) receives a copy of the status header so the host can read it
// without a copy launch.
template <int NT>
__device__ void schedule_block(const vs_config& cfg, const vs_state& st, int N, int first, int do_remove,
                               int admit_mode, int select_mode, int32_t* mirror, int* smem) {
  const int tid = threadIdx.x;
  const int n = cfg.n, k = cfg.k;
  int* live_s = smem;
  int* order_s = live_s + n;
  int* tmp_s = order_s + n;
  int* flags_s = tmp_s + n;
  int* lt_s = flags_s + n;
  int* act_s = lt_s + n;
  int* input_s = act_s + n;
  int* width_s = input_s + n;
  int* off_s = width_s + n;  // [n + 1]
  int* sh = off_s + n + 1;   // [8] block-uniform results, then [32] scan partials
  int32_t* status = st.status;
  int32_t* stat_sel = status + VS_ST_HDR;
  int32_t* stat_fin = stat_sel + n;
  int32_t* stat_live = stat_fin + n;
  int32_t* stat_adm = stat_live + n;

  // ---- one round of independent loads (all threads) -------------------------------
  // __ldcg: L2-coherent loads — in the fused kernel other CTAs wrote this state
  // after this SM may have cached neighbouring lines in L1
  for (int i = tid; i < n; i += NT) {
    flags_s[i] = first ? 0 : __ldcg(&st.slot_flags[i]);
    lt_s[i] = __ldcg(&st.slot_lt[i]);
    act_s[i] = __ldcg(&st.slot_active[i]);
    width_s[i] = __ldcg(&st.slot_width[i]);
    input_s[i] = __ldcg(&st.slot_input[i]);
    live_s[i] = __ldcg(&st.live[i]);
    order_s[i] = first ? 0 : __ldcg(&st.sel[i]);  // previous selection (for finished ids)
  }
  __syncthreads();
  VS_PROF(true, 9);

  // ===== phases A-C, all NT threads: thread t owns the contiguous items
  // [t*ipt, t*ipt + ipt); every stable compaction is one block scan of
  // per-thread counts (a handful of barriers instead of one warp's long
  // dependent chain of loops over n / 32 items per lane) =====================
  const int sticky = first ? 0 : __ldcg(&st.counters[3]);  // contract error from the beam step
  int n_live = first ? 0 : __ldcg(&st.counters[0]);
  int cursor = first ? 0 : __ldcg(&st.counters[1]);
  const int nsel_prev = first ? 0 : __ldcg(&status[VS_ST_NSEL]);
  const int ipt = (n + NT - 1) / NT;
  const int i0 = min(n, tid * ipt), i1 = min(n, i0 + ipt);
  int* wsum = sh + 8;  // [NT / 32] block-scan partials
  int tot;
  VS_PROF(true, 12);

  // ---- A. removal of finished beams (stable) ----------------------------------------
  int nfin = 0;
  if (do_remove && !first) {
    int c = 0;  // finished ids in selection order (bb/scheduler.py:186-189)
    #pragma unroll 1
    for (int i = i0; i < min(i1, nsel_prev); ++i) c += (flags_s[order_s[i]] & 2) != 0;
    int p = block_excl_scan<NT>(c, wsum, &nfin);
    #pragma unroll 1
    for (int i = i0; i < min(i1, nsel_prev); ++i) {
      const int s = order_s[i];
      if (flags_s[s] & 2) stat_fin[p++] = input_s[s];
    }
    c = 0;
    #pragma unroll 1
    for (int i = i0; i < min(i1, n_live); ++i) c += !(flags_s[live_s[i]] & 2);
    p = block_excl_scan<NT>(c, wsum, &tot);
    #pragma unroll 1
    for (int i = i0; i < min(i1, n_live); ++i) {  // each live slot is owned by one thread
      const int s = live_s[i];
      if (!(flags_s[s] & 2)) tmp_s[p++] = s;
      else flags_s[s] = 0;  // slot freed
    }
    n_live = tot;
    __syncthreads();
    for (int i = tid; i < n_live; i += NT) live_s[i] = tmp_s[i];
    __syncthreads();
  }
  const int n_live_after = n_live;
  VS_PROF(true, 13);
  for (int i = tid; i < n_live_after; i += NT) stat_live[i] = input_s[live_s[i]];

  // ---- B. refill --------------------------------------------------------------------
  int n_admit = 0;
  const int admit0 = cursor;
  bool admit = false;
  if (cursor < N) {
    if (admit_mode == VS_ADMIT_VARSTREAM) admit = n_live <= cfg.refill_threshold;
    else if (admit_mode == VS_ADMIT_VARBEAM) admit = n_live == 0;
    else if (admit_mode == VS_ADMIT_VARFIFO) admit = n_live < n;
  }
  if (admit) {
    n_admit = min(n - n_live, N - cursor);
    int c = 0;
    #pragma unroll 1
    for (int s = i0; s < i1; ++s) c += !(flags_s[s] & 1);
    int fpos = block_excl_scan<NT>(c, wsum, &tot);
    #pragma unroll 1
    for (int s = i0; s < i1; ++s) {  // the n_admit lowest free slots, ascending
      if (flags_s[s] & 1) continue;
      if (fpos < n_admit) tmp_s[fpos] = s;
      ++fpos;
    }
    __syncthreads();
    // admitted slot q takes input cursor + q
    for (int q = tid; q < n_admit; q += NT) {
      const int s = tmp_s[q], input = cursor + q;
      const int so0 = st.src_off[input], so1 = st.src_off[input + 1];
      live_s[n_live + q] = s;
      stat_adm[q] = s;
      flags_s[s] = 1;
      input_s[s] = input;
      lt_s[s] = 1;  // Beam.initial, bb/core.py:79-82
      act_s[s] = 1;
      width_s[s] = 1;
      st.slot_input[s] = input;
      st.slot_lt[s] = 1;
      st.slot_emitted[s] = 0;
      st.slot_width[s] = 1;
      st.slot_active[s] = 1;
      st.slot_src_len[s] = so1 - so0;
      st.c_score[s * k] = 0.0;
      st.c_len[s * k] = 1;
      st.c_row[s * k] = 0;
      st.c_fin[s * k] = 0;
      st.c_hash[s * k] = 0;
      st.c_act[s * k] = act_pack(0, 0);
      st.hist[(int64_t)(s * k) * cfg.max_len] = cfg.sos;
      st.out_count[input] = 0;
    }
    n_live += n_admit;
    cursor += n_admit;
    __syncthreads();
  }
  for (int i = tid; i < n; i += NT) st.slot_flags[i] = flags_s[i];
  VS_PROF(true, 10);

  // ---- C. selection -------------------------------------------------------------------
  int nc = 0, eff = 0;
  if (n_live > 0) {
    const int j1 = min(i1, n_live);
    if (select_mode == VS_SELECT_MIN_LT) {
      int lmin = 0x7fffffff;
      #pragma unroll 1
      for (int i = i0; i < j1; ++i) lmin = min(lmin, lt_s[live_s[i]]);
      eff = block_min<NT>(lmin, wsum);
      int c = 0;
      #pragma unroll 1
      for (int i = i0; i < j1; ++i) c += lt_s[live_s[i]] == eff;
      int p = block_excl_scan<NT>(c, wsum, &nc);
      #pragma unroll 1
      for (int i = i0; i < j1; ++i) {
        const int s = live_s[i];
        if (lt_s[s] == eff) order_s[p++] = s;
      }
    } else if (select_mode == VS_SELECT_FIFO) {  // sort by (-l_t, arrival)
      for (int i = tid; i < n_live; i += NT) {
        const int s = live_s[i], lt = lt_s[s];
        int rank = 0;
        #pragma unroll 1
        for (int q = 0; q < n_live; ++q) {
          const int lq = lt_s[live_s[q]];
          rank += (lq > lt) || (lq == lt && q < i);
        }
        order_s[rank] = s;
      }
      nc = n_live;
    } else {
      for (int i = tid; i < n_live; i += NT) order_s[i] = live_s[i];
      nc = n_live;
    }
    __syncthreads();
  }

  // pack (bb/scheduler.py:119-132): fast path when everything fits
  int wsum_l = 0, bad_l = 0;
  const int k1 = min(i1, nc);
  #pragma unroll 1
  for (int i = i0; i < k1; ++i) {
    const int wd = act_s[order_s[i]];
    wsum_l += wd;
    bad_l |= wd > cfg.capacity;
  }
  int tot_w;
  int wpos = block_excl_scan<NT>(wsum_l, wsum, &tot_w);
  const int bad = __syncthreads_or(bad_l);
  int nsel = 0, R = 0;
  if (!bad && tot_w <= cfg.capacity) {
    #pragma unroll 1
    for (int i = i0; i < k1; ++i) {
      const int s = order_s[i];
      st.sel[i] = s;
      st.sel_off[i] = wpos;
      off_s[i] = wpos;
      wpos += act_s[s];
    }
    nsel = nc;
    R = tot_w;
  } else if (!bad) {
    if (tid == 0) {
      int total = 0, c = 0;
      #pragma unroll 1
      for (int i = 0; i < nc; ++i) {
        const int s = order_s[i];
        const int wi = act_s[s];
        if (total + wi <= cfg.capacity) {
          order_s[c] = s;  // in place: c <= i
          st.sel[c] = s;
          st.sel_off[c] = total;
          off_s[c] = total;
          ++c;
          total += wi;
        }
      }
      sh[2] = c;
      sh[3] = total;
    }
    __syncthreads();
    nsel = sh[2];
    R = sh[3];
  }
  if (select_mode != VS_SELECT_MIN_LT && nsel > 0) {  // effective_len = max l_t of chosen
    int m = 0x7fffffff;
    #pragma unroll 1
    for (int i = i0; i < min(i1, nsel); ++i) m = min(m, -lt_s[order_s[i]]);
    eff = -block_min<NT>(m, wsum);
  }
  if (n_live == 0) eff = 0;
  __syncthreads();  // order_s / off_s complete
  for (int i = tid; i < nsel; i += NT) stat_sel[i] = input_s[order_s[i]];
  for (int i = tid; i < n_live; i += NT) st.live[i] = live_s[i];
  if (tid == 0) {
    st.sel_off[nsel] = R;
    off_s[nsel] = R;
    sh[0] = nsel;
    sh[1] = R;
    int hdr[VS_ST_HDR] = {};
    hdr[VS_ST_R] = R;
    hdr[VS_ST_NSEL] = nsel;
    hdr[VS_ST_NLIVE] = n_live;
    hdr[VS_ST_L] = eff;
    hdr[VS_ST_NADMIT] = n_admit;
    hdr[VS_ST_ADMIT0] = admit0;
    hdr[VS_ST_CURSOR] = cursor;
    hdr[VS_ST_DONE] = (n_live == 0) ? 1 : 0;
    hdr[VS_ST_ERROR] = bad ? VS_ERR_CONFIG : sticky;
    hdr[VS_ST_NFIN] = nfin;
    hdr[VS_ST_NLIVE_AFTER] = n_live_after;
    const int fill = first ? 0 : __ldcg(&st.counters[6]);
    hdr[VS_ST_TOKFILL] = fill;
    // arrival order == input order and removal is stable: live[0] is the
    // oldest live input, and every input below it has finished
    hdr[VS_ST_MINLIVE] = n_live > 0 ? input_s[live_s[0]] : cursor;
#pragma unroll
    for (int q = 0; q < VS_ST_HDR; ++q) status[q] = hdr[q];
    // the host reads the mirror after an event recorded behind this kernel:
    // kernel completion makes these writes visible, no system fence needed
    if (mirror) {
#pragma unroll
      for (int q = 0; q < VS_ST_HDR; ++q) mirror[q] = hdr[q];
    }
    st.counters[0] = n_live;
    st.counters[1] = cursor;
    st.counters[2] = N;
    st.counters[3] = sticky;
    st.counters[6] = fill;
  }
  __syncthreads();
  VS_PROF(true, 11);

  // ---- D. row list (all threads): r -> (beam by binary search over off_s, ordinal) --
  constexpr int UNR = 4;
  for (int r0 = 0; r0 < R; r0 += NT * UNR) {
    int pk[UNR], sl[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int r = r0 + u * NT + tid;
      sl[u] = -1;
      if (r < R) {
        int lo = 0, hi = nsel - 1;  // last beam b with off_s[b] <= r
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (off_s[mid] <= r) lo = mid;
          else hi = mid - 1;
        }
        const int s = order_s[lo];
        sl[u] = s;
        pk[u] = __ldcg(&st.c_act[s * k + (r - off_s[lo])]);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int r = r0 + u * NT + tid;
      if (sl[u] >= 0) {
        const int s = sl[u];
        st.row_slot[r] = s;
        st.row_cand[r] = pk[u] & 0xff;
        st.row_phys[r] = s * k + (pk[u] >> 8);
        st.row_len[r] = lt_s[s];  // every active candidate of a beam has length l_t
      }
    }
  }
}

}  // namespace vs
