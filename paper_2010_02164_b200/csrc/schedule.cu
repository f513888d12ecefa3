// K3 compact_refill_select: the VarStream scheduler step on device (sm_100a).
//
// One CTA (1024 threads, one live-list entry per thread) per call:
//   A. stable removal of finished beams      bb/scheduler.py:190-192 (+ finished
//      ids in selection order :186-189 for StepEvent)
//   B. ε-refill at the top of the step        bb/scheduler.py:94-116, :237-240,
//      admit predicates :306 / :335 / :359, checked once (:266-268)
//   C. selection with capacity packing       bb/scheduler.py:119-165
//      (min-l_t in arrival order / FIFO most-advanced first / all for flush;
//      greedy arrival-order fill, skip and continue; width > capacity ->
//      ConfigError :125-128)
//   D. the next step's row list: active candidates of the selected beams in
//      beam order (bb/search.py:223-225)
// Slots never move: the live list is an index list and admission takes the
// lowest free slot ids (physical placement does not affect results).
#include "common.cuh"

namespace vs {
namespace {

constexpr int NT3 = 1024;

// Block-wide exclusive scan of one int per thread; returns exclusive prefix, total in *tot.
__device__ int block_excl_scan(int v, int* warp_sums, int* tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < (NT3 / 32) ? warp_sums[lane] : 0;
    int incl = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    warp_sums[lane] = incl - w;  // exclusive warp offsets
    if (lane == 31) warp_sums[32] = incl;
  }
  __syncthreads();
  const int res = warp_sums[wid] + x - v;
  *tot = warp_sums[32];
  __syncthreads();
  return res;
}

__global__ void __launch_bounds__(NT3) schedule_kernel(vs_config cfg, vs_state st, int N, int first,
                                                       int do_remove, int admit_mode, int select_mode) {
  __shared__ int wsum[33];
  __shared__ int live_s[VS_MAX_SLOTS];
  __shared__ int order_s[VS_MAX_SLOTS];
  __shared__ int sh[16];
  const int tid = threadIdx.x;
  const int n = cfg.n, k = cfg.k;
  int32_t* status = st.status;
  int32_t* stat_sel = status + VS_ST_HDR;
  int32_t* stat_fin = stat_sel + n;
  int32_t* stat_live = stat_fin + n;
  int32_t* stat_adm = stat_live + n;

  if (first) {
    for (int s = tid; s < n; s += NT3) st.slot_flags[s] = 0;
    if (tid == 0) {
      st.counters[0] = 0;
      st.counters[1] = 0;
      st.counters[2] = N;
      status[VS_ST_NSEL] = 0;
    }
    __syncthreads();
  }
  int n_live = st.counters[0];
  int cursor = st.counters[1];
  if (tid < n_live) live_s[tid] = st.live[tid];
  if (tid == 0) {
    sh[0] = 0;  // nfin
    sh[1] = 0;  // error
  }
  __syncthreads();

  // ---- A. removal of finished beams (stable) ------------------------------------
  if (do_remove && !first) {
    {  // finished ids in selection order (bb/scheduler.py:186-189), parallel
      const int nsel_prev = status[VS_ST_NSEL];
      int f = 0, fin_input = 0;
      if (tid < nsel_prev) {
        const int s = st.sel[tid];
        f = (st.slot_flags[s] & 2) != 0;
        if (f) fin_input = st.slot_input[s];
      }
      int tot;
      const int p = block_excl_scan(f, wsum, &tot);
      if (f) stat_fin[p] = fin_input;
      if (tid == 0) sh[0] = tot;
    }
    int s = -1, keep = 0;
    if (tid < n_live) {
      s = live_s[tid];
      keep = !(st.slot_flags[s] & 2);
    }
    int tot;
    const int pos = block_excl_scan(keep, wsum, &tot);
    __syncthreads();
    if (tid < n_live) {
      if (keep) live_s[pos] = s;
      else st.slot_flags[s] = 0;  // slot freed
    }
    n_live = tot;
    __syncthreads();
  }
  const int n_live_after = n_live;
  if (tid < n_live_after) stat_live[tid] = st.slot_input[live_s[tid]];

  // ---- B. refill ------------------------------------------------------------------------
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
    int is_free = 0, s = tid;
    if (tid < n) is_free = !(st.slot_flags[s] & 1);
    int tot;
    const int fpos = block_excl_scan(is_free, wsum, &tot);
    if (is_free && fpos < n_admit) {
      const int input = cursor + fpos;
      live_s[n_live + fpos] = s;
      stat_adm[fpos] = s;
      st.slot_flags[s] = 1;
      st.slot_input[s] = input;
      st.slot_lt[s] = 1;  // Beam.initial, bb/core.py:79-82
      st.slot_emitted[s] = 0;
      st.slot_width[s] = 1;
      st.slot_active[s] = 1;
      st.slot_src_len[s] = st.src_off[input + 1] - st.src_off[input];
      st.c_score[s * k] = 0.0;
      st.c_len[s * k] = 1;
      st.c_row[s * k] = 0;
      st.c_fin[s * k] = 0;
      st.c_hash[s * k] = 0;
      st.hist[(int64_t)(s * k) * cfg.max_len] = cfg.sos;
      st.out_count[input] = 0;
    }
    n_live += n_admit;
    cursor += n_admit;
    __syncthreads();
  }

  // ---- C. selection -------------------------------------------------------------------
  // candidate list in advance order -> order_s[0..nc)
  int nc = 0;
  int eff = 0;
  if (n_live > 0) {
    int lt = 0, s = -1;
    if (tid < n_live) {
      s = live_s[tid];
      lt = st.slot_lt[s];
    }
    if (select_mode == VS_SELECT_MIN_LT) {
      int mn = tid < n_live ? lt : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      if ((tid & 31) == 0) order_s[tid >> 5] = mn;
      __syncthreads();
      if (tid == 0) {
        int m = 0x7fffffff;
        for (int wv = 0; wv < NT3 / 32; ++wv) m = min(m, order_s[wv]);
        sh[2] = m;
      }
      __syncthreads();
      eff = sh[2];
      const int in_front = tid < n_live && lt == eff;
      int tot;
      const int p = block_excl_scan(in_front, wsum, &tot);
      if (in_front) order_s[p] = s;
      nc = tot;
    } else if (select_mode == VS_SELECT_FIFO) {  // sort by (-l_t, arrival)
      if (tid < n_live) {
        int rank = 0;
        for (int j = 0; j < n_live; ++j) {
          const int lj = st.slot_lt[live_s[j]];
          rank += (lj > lt) || (lj == lt && j < tid);
        }
        order_s[rank] = s;
      }
      nc = n_live;
    } else {
      if (tid < n_live) order_s[tid] = s;
      nc = n_live;
    }
    __syncthreads();
  }

  // pack (bb/scheduler.py:119-132): fast path when everything fits
  int w = 0;
  if (tid < nc) w = st.slot_active[order_s[tid]];
  int tot_w;
  const int wpos = block_excl_scan(w, wsum, &tot_w);
  int nsel = 0, R = 0;
  int bad = __syncthreads_or(tid < nc && w > cfg.capacity);
  if (bad) {
    if (tid == 0) sh[1] = VS_ERR_CONFIG;
  } else if (tot_w <= cfg.capacity) {
    if (tid < nc) {
      st.sel[tid] = order_s[tid];
      st.sel_off[tid] = wpos;
    }
    nsel = nc;
    R = tot_w;
  } else {
    if (tid == 0) {
      int total = 0, c = 0;
      for (int i = 0; i < nc; ++i) {
        const int s = order_s[i];
        const int wi = st.slot_active[s];
        if (total + wi <= cfg.capacity) {
          st.sel[c] = s;
          st.sel_off[c] = total;
          ++c;
          total += wi;
        }
      }
      sh[3] = c;
      sh[4] = total;
    }
    __syncthreads();
    nsel = sh[3];
    R = sh[4];
  }
  if (tid == 0) st.sel_off[nsel] = R;
  __syncthreads();
  if (select_mode != VS_SELECT_MIN_LT && nsel > 0) {  // effective_len = max l_t of chosen
    int lt = tid < nsel ? st.slot_lt[st.sel[tid]] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lt = max(lt, __shfl_xor_sync(0xffffffffu, lt, o));
    if ((tid & 31) == 0) wsum[tid >> 5] = lt;
    __syncthreads();
    if (tid == 0) {
      int m = 0;
      for (int wv = 0; wv < NT3 / 32; ++wv) m = max(m, wsum[wv]);
      sh[5] = m;
    }
    __syncthreads();
    eff = sh[5];
  }
  if (n_live == 0) eff = 0;

  // ---- D. row list: active candidates of each selected beam, beam order ------------
  // one warp per selected beam: ballot-compact its active candidates (beam order)
  {
    const int lane = tid & 31, wid = tid >> 5;
    for (int b = wid; b < nsel; b += NT3 / 32) {
      const int s = st.sel[b];
      const int r0 = st.sel_off[b];
      const int width = st.slot_width[s];
      int before = 0;
      for (int j0 = 0; j0 < width; j0 += 32) {
        const int j = j0 + lane;
        const int c = s * k + j;
        const bool act = j < width && !st.c_fin[c];
        const unsigned m = __ballot_sync(0xffffffffu, act);
        if (act) {
          const int r = r0 + before + __popc(m & ((1u << lane) - 1u));
          st.row_slot[r] = s;
          st.row_cand[r] = j;
          st.row_phys[r] = s * k + st.c_row[c];
          st.row_len[r] = st.c_len[c];
        }
        before += __popc(m);
      }
      if (lane == 0) stat_sel[b] = st.slot_input[s];
    }
  }
  if (tid < n_live) st.live[tid] = live_s[tid];
  if (tid == 0) {
    status[VS_ST_R] = R;
    status[VS_ST_NSEL] = nsel;
    status[VS_ST_NLIVE] = n_live;
    status[VS_ST_L] = eff;
    status[VS_ST_NADMIT] = n_admit;
    status[VS_ST_ADMIT0] = admit0;
    status[VS_ST_CURSOR] = cursor;
    status[VS_ST_DONE] = (n_live == 0) ? 1 : 0;
    status[VS_ST_ERROR] = sh[1];
    status[VS_ST_NFIN] = sh[0];
    status[VS_ST_NLIVE_AFTER] = n_live_after;
    st.counters[0] = n_live;
    st.counters[1] = cursor;
    *st.n_copy = 0;
  }
}

}  // namespace
}  // namespace vs

extern "C" int vs_schedule(const vs_config* cfg, const vs_state* st, int32_t N, int32_t first_call,
                           int32_t do_remove, int32_t admit_mode, int32_t select_mode, void* stream) {
  if (!cfg || !st || cfg->n < 1 || cfg->n > VS_MAX_SLOTS || cfg->k < 1 || cfg->k > VS_MAX_K ||
      N < 1 || cfg->capacity < cfg->k)
    return VS_ERR_CONFIG;
  vs::schedule_kernel<<<1, vs::NT3, 0, static_cast<cudaStream_t>(stream)>>>(
      *cfg, *st, N, first_call, do_remove, admit_mode, select_mode);
  VS_CUDA_RET();
}
