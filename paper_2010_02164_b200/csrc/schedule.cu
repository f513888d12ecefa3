// K3 compact_refill_select: the VarStream scheduler step on device (sm_100a).
//
// One CTA (1024 threads, one slot / live-list entry per thread) per call:
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
// All per-slot state is pulled into shared memory in one round of independent
// loads, so the kernel costs ~3 dependent global round trips.  Slots never
// move: the live list is an index list and admission takes the lowest free
// slot ids (physical placement does not affect results).
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

__device__ __forceinline__ int block_min(int v, int* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  int m = 0x7fffffff;
  for (int q = 0; q < NT3 / 32; ++q) m = min(m, scratch[q]);
  __syncthreads();
  return m;
}

__global__ void __launch_bounds__(NT3) schedule_kernel(vs_config cfg, vs_state st, int N, int first,
                                                       int do_remove, int admit_mode, int select_mode) {
  VS_PDL_ENTRY();
  __shared__ int wsum[33];
  __shared__ int live_s[VS_MAX_SLOTS];
  __shared__ int order_s[VS_MAX_SLOTS];
  __shared__ int flags_s[VS_MAX_SLOTS], lt_s[VS_MAX_SLOTS], act_s[VS_MAX_SLOTS], input_s[VS_MAX_SLOTS];
  __shared__ int width_s[VS_MAX_SLOTS], off_s[VS_MAX_SLOTS + 1];
  __shared__ int sh[8];
  const int tid = threadIdx.x;
  const int n = cfg.n, k = cfg.k;
  int32_t* status = st.status;
  int32_t* stat_sel = status + VS_ST_HDR;
  int32_t* stat_fin = stat_sel + n;
  int32_t* stat_live = stat_fin + n;
  int32_t* stat_adm = stat_live + n;

  // ---- one round of independent loads -------------------------------------------
  const int sticky = first ? 0 : st.counters[3];  // device contract error from beam_step
  int n_live = first ? 0 : st.counters[0];
  int cursor = first ? 0 : st.counters[1];
  const int nsel_prev = first ? 0 : status[VS_ST_NSEL];
  int prev_sel = -1;
  if (tid < n) {
    flags_s[tid] = first ? 0 : st.slot_flags[tid];
    lt_s[tid] = st.slot_lt[tid];
    act_s[tid] = st.slot_active[tid];
    width_s[tid] = st.slot_width[tid];
    input_s[tid] = st.slot_input[tid];
    live_s[tid] = st.live[tid];
    prev_sel = st.sel[tid];
  }
  __syncthreads();

  // ---- A. removal of finished beams (stable) ------------------------------------
  int nfin = 0;
  if (do_remove && !first) {
    {  // finished ids in selection order (bb/scheduler.py:186-189)
      int f = 0, fin_input = 0;
      if (tid < nsel_prev) {
        f = (flags_s[prev_sel] & 2) != 0;
        if (f) fin_input = input_s[prev_sel];
      }
      int tot;
      const int p = block_excl_scan(f, wsum, &tot);
      if (f) stat_fin[p] = fin_input;
      nfin = tot;
    }
    int s = -1, keep = 0;
    if (tid < n_live) {
      s = live_s[tid];
      keep = !(flags_s[s] & 2);
    }
    int tot;
    const int pos = block_excl_scan(keep, wsum, &tot);
    if (tid < n_live) {
      if (keep) live_s[pos] = s;
      else flags_s[s] = 0;  // slot freed
    }
    n_live = tot;
    __syncthreads();
  }
  const int n_live_after = n_live;
  if (tid < n_live_after) stat_live[tid] = input_s[live_s[tid]];

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
    const int is_free = tid < n && !(flags_s[tid] & 1);
    int tot;
    const int fpos = block_excl_scan(is_free, wsum, &tot);
    if (is_free && fpos < n_admit) {
      const int s = tid, input = cursor + fpos;
      live_s[n_live + fpos] = s;
      stat_adm[fpos] = s;
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
  if (tid < n) st.slot_flags[tid] = flags_s[tid];

  // ---- C. selection -------------------------------------------------------------------
  int nc = 0, eff = 0;
  if (n_live > 0) {
    int lt = 0x7fffffff, s = -1;
    if (tid < n_live) {
      s = live_s[tid];
      lt = lt_s[s];
    }
    if (select_mode == VS_SELECT_MIN_LT) {
      eff = block_min(lt, wsum);
      const int in_front = tid < n_live && lt == eff;
      int tot;
      const int p = block_excl_scan(in_front, wsum, &tot);
      if (in_front) order_s[p] = s;
      nc = tot;
    } else if (select_mode == VS_SELECT_FIFO) {  // sort by (-l_t, arrival)
      if (tid < n_live) {
        int rank = 0;
        for (int q = 0; q < n_live; ++q) {
          const int lq = lt_s[live_s[q]];
          rank += (lq > lt) || (lq == lt && q < tid);
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
  const int wdt = tid < nc ? act_s[order_s[tid]] : 0;
  int tot_w;
  const int wpos = block_excl_scan(wdt, wsum, &tot_w);
  int nsel = 0, R = 0;
  const int bad = __syncthreads_or(tid < nc && wdt > cfg.capacity);
  if (!bad && tot_w <= cfg.capacity) {
    if (tid < nc) {
      st.sel[tid] = order_s[tid];
      st.sel_off[tid] = wpos;
      off_s[tid] = wpos;
    }
    nsel = nc;
    R = tot_w;
  } else if (!bad) {
    if (tid == 0) {
      int total = 0, c = 0;
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
      sh[3] = c;
      sh[4] = total;
    }
    __syncthreads();
    nsel = sh[3];
    R = sh[4];
  }
  if (tid == 0) st.sel_off[nsel] = R;
  if (select_mode != VS_SELECT_MIN_LT && nsel > 0)  // effective_len = max l_t of chosen
    eff = -block_min(tid < nsel ? -lt_s[order_s[tid]] : 0x7fffffff, wsum);
  if (n_live == 0) eff = 0;

  // ---- D. row list: active candidates of each selected beam, beam order ------------
  // one warp per selected beam; a warp's (<= 4 beams) x (<= 2 chunks of 32)
  // candidate loads are issued together so the phase costs one round trip.
  __syncthreads();
  {
    const int lane = tid & 31, wid = tid >> 5;
    constexpr int NB = VS_MAX_SLOTS / (NT3 / 32) > 4 ? 4 : VS_MAX_SLOTS / (NT3 / 32);
    if (k <= 64 && nsel <= NB * (NT3 / 32)) {
      unsigned char fz[NB][2];
      int rw[NB][2], ln[NB][2];
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int b = wid + 32 * i;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          fz[i][h] = 1;
          if (b < nsel) {
            const int sb = order_s[b];
            const int j = 32 * h + lane;
            if (j < width_s[sb]) {
              const int c = sb * k + j;
              fz[i][h] = st.c_fin[c];
              rw[i][h] = st.c_row[c];
              ln[i][h] = st.c_len[c];
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int b = wid + 32 * i;
        if (b >= nsel) break;
        const int sb = order_s[b];
        int r = off_s[b];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bool a = !fz[i][h];
          const unsigned m = __ballot_sync(0xffffffffu, a);
          if (a) {
            const int rr = r + __popc(m & ((1u << lane) - 1u));
            st.row_slot[rr] = sb;
            st.row_cand[rr] = 32 * h + lane;
            st.row_phys[rr] = sb * k + rw[i][h];
            st.row_len[rr] = ln[i][h];
          }
          r += __popc(m);
        }
        if (lane == 0) stat_sel[b] = input_s[sb];
      }
    } else {  // generic path (k > 64 or very large n)
      for (int b = wid; b < nsel; b += NT3 / 32) {
        const int sb = order_s[b];
        int r = off_s[b];
        for (int j0 = 0; j0 < width_s[sb]; j0 += 32) {
          const int j = j0 + lane;
          const int c = sb * k + j;
          const bool a = j < width_s[sb] && !st.c_fin[c];
          const unsigned m = __ballot_sync(0xffffffffu, a);
          if (a) {
            const int rr = r + __popc(m & ((1u << lane) - 1u));
            st.row_slot[rr] = sb;
            st.row_cand[rr] = j;
            st.row_phys[rr] = sb * k + st.c_row[c];
            st.row_len[rr] = st.c_len[c];
          }
          r += __popc(m);
        }
        if (lane == 0) stat_sel[b] = input_s[sb];
      }
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
    status[VS_ST_ERROR] = bad ? VS_ERR_CONFIG : sticky;
    status[VS_ST_NFIN] = nfin;
    status[VS_ST_NLIVE_AFTER] = n_live_after;
    st.counters[0] = n_live;
    st.counters[1] = cursor;
    st.counters[2] = N;
    st.counters[3] = sticky;
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
  vs::vs_launch(vs::schedule_kernel, dim3(1), dim3(vs::NT3), 0, static_cast<cudaStream_t>(stream), 
      *cfg, *st, N, first_call, do_remove, admit_mode, select_mode);
  VS_CUDA_RET();
}
