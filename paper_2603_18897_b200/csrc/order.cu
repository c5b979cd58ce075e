// K1 general path: ingest_trace's grouping, stable (t_start, seq) sort,
// reorder tally and inactivity split (events.py:196-252) over a columnar
// trace in arrival order, on the device.
//
//   1. order_count_kernel   events per session id, tool events per id,
//                           "grouped?" (ids non-decreasing), NaN t_start;
//                           warp-aggregated atomics (__match_any_sync), so a
//                           grouped trace costs one atomic per run of a
//                           session inside a warp
//   2. exclusive scans      event offsets and tool offsets per session
//   3. order_place_kernel   interleaved traces only: scatter arrival indices
//                           into their session's range (any order inside it:
//                           the sort's last key is the arrival index, so the
//                           result is the stable order regardless)
//   4. order_warp_kernel    one warp per session of <= 32 events: registers +
//                           shuffles (sortedness probe, 32-lane bitonic sort
//                           only when needed), reorder check against the
//                           arrival-order seq list, gap split, tool ranks,
//                           output written in place
//   5. order_cta_kernel     one CTA per longer session: shared-memory bitonic
//                           chunks + merge-path passes in global scratch;
//                           interleaved sessions are first sorted by arrival
//                           to recover the arrival-order seq list
//   6. segment numbering    scan of segments per session, then a warp per
//                           session adds its base to its tool events
//
// The trace stays in HBM: for a grouped, already-sorted trace the traffic is
// the 28 B/event column read plus the 28 B/event write of the tool events
// and the small per-session arrays.
#include <algorithm>

#include "common.cuh"

namespace paste {
namespace {

constexpr int OT = 256;           // threads: count / place / scan / warp kernels
constexpr int SCAN_IPT = 8;
constexpr int SCAN_TILE = OT * SCAN_IPT;
constexpr int CT = 512;           // CTA sort threads
constexpr int CHUNK = 2048;       // CTA sort shared-memory chunk (elements)
constexpr int MIPT = 8;           // merge outputs per thread per step

struct OKey {
  double t;
  int32_t seq;
  int32_t arr;
};

struct OrderCounters {
  unsigned long long ungrouped, bad_session, nan_t, n_big, reordered;
};

__device__ __forceinline__ double norm_t(double t) { return t == 0.0 ? 0.0 : t; }  // -0.0 == 0.0

template <int MODE>  // 0: by arrival; 1: by (t_start, seq, arrival)
__device__ __forceinline__ bool okey_less(const OKey& a, const OKey& b) {
  if (MODE == 0) return a.arr < b.arr;
  if (a.t != b.t) return a.t < b.t;
  if (a.seq != b.seq) return a.seq < b.seq;
  return a.arr < b.arr;
}

__device__ __forceinline__ OKey sentinel() {
  OKey k;
  k.t = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  k.seq = INT32_MAX;
  k.arr = INT32_MAX;
  return k;
}

__device__ __forceinline__ OKey shfl_key(const OKey& k, int src) {
  OKey o;
  o.t = __shfl_sync(0xffffffffu, k.t, src);
  o.seq = __shfl_sync(0xffffffffu, k.seq, src);
  o.arr = __shfl_sync(0xffffffffu, k.arr, src);
  return o;
}

__device__ __forceinline__ OKey shfl_xor_key(const OKey& k, int m) {
  OKey o;
  o.t = __shfl_xor_sync(0xffffffffu, k.t, m);
  o.seq = __shfl_xor_sync(0xffffffffu, k.seq, m);
  o.arr = __shfl_xor_sync(0xffffffffu, k.arr, m);
  return o;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------
// 1. counts
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(OT) order_count_kernel(const paste_order_desc d, int32_t* cnt,
                                                         int32_t* ntool, OrderCounters* c) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * OT;
  unsigned long long ung = 0, bad = 0, nan = 0;
  for (int64_t base = (int64_t)blockIdx.x * OT; base < d.n_events; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool v = i < d.n_events;
    int32_t s = v ? d.session[i] : -1;
    const bool ok = v && (uint32_t)s < (uint32_t)d.n_sessions;
    if (v && !ok) ++bad;
    if (v) {
      const double t = d.t_start[i];
      if (t != t) ++nan;
      if (i > 0 && d.session[i - 1] > s) ++ung;
    }
    const bool tool = ok && d.sig[i] >= 0;
    const int key = ok ? s : -1 - lane;  // invalid lanes never group
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const unsigned tools = peers & __ballot_sync(0xffffffffu, tool);
    if (ok && lane == __ffs(peers) - 1) {
      atomicAdd(&cnt[s], __popc(peers));
      if (tools) atomicAdd(&ntool[s], __popc(tools));
    }
  }
  if (ung) atomicAdd(&c->ungrouped, ung);
  if (bad) atomicAdd(&c->bad_session, bad);
  if (nan) atomicAdd(&c->nan_t, nan);
}

// ---------------------------------------------------------------------------
// 2. exclusive scan int32[n] -> int64[n + 1] (three launches)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* total) {
  __shared__ int64_t warp_tot[OT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t t = lane < OT / 32 ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < OT / 32) warp_tot[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  const int64_t wbase = w ? warp_tot[w - 1] : 0;
  *total = warp_tot[OT / 32 - 1];
  __syncthreads();
  return wbase + x - v;
}

__global__ void __launch_bounds__(OT) scan_reduce_kernel(const int32_t* in, int64_t n,
                                                         int64_t* bsum) {
  const int64_t t0 = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    const int64_t i = t0 + (int64_t)k * OT + threadIdx.x;
    if (i < n) s += in[i];
  }
  int64_t tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(OT) scan_bsums_kernel(int64_t* bsum, int64_t nb, int64_t* out,
                                                        int64_t n) {
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += OT) {
    const int64_t b = b0 + threadIdx.x;
    const int64_t v = b < nb ? bsum[b] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan(v, &tot);
    if (b < nb) bsum[b] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) out[n] = carry;
}

__global__ void __launch_bounds__(OT) scan_down_kernel(const int32_t* in, int64_t n,
                                                       const int64_t* bsum, int64_t* out) {
  // thread t owns SCAN_IPT consecutive elements of the tile
  const int64_t t0 = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
  int32_t v[SCAN_IPT];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    v[k] = t0 + k < n ? in[t0 + k] : 0;
    s += v[k];
  }
  int64_t tot;
  int64_t run = bsum[blockIdx.x] + block_excl_scan(s, &tot);
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    if (t0 + k < n) out[t0 + k] = run;
    run += v[k];
  }
}

int scan_i32(const int32_t* in, int64_t* out, int64_t n, int64_t* bsum, cudaStream_t st) {
  const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (nb > 0) {
    scan_reduce_kernel<<<(unsigned)nb, OT, 0, st>>>(in, n, bsum);
  }
  scan_bsums_kernel<<<1, OT, 0, st>>>(bsum, nb, out, n);
  if (nb > 0) scan_down_kernel<<<(unsigned)nb, OT, 0, st>>>(in, n, bsum, out);
  count_launch(nb > 0 ? 3 : 1);
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

// ---------------------------------------------------------------------------
// 3. placement of interleaved traces
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(OT) order_place_kernel(const paste_order_desc d,
                                                         const int64_t* off, int32_t* cursor,
                                                         int32_t* perm, const OrderCounters* c) {
  if (c->ungrouped == 0 || c->bad_session != 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * OT;
  for (int64_t base = (int64_t)blockIdx.x * OT; base < d.n_events; base += stride) {
    const int64_t i = base + threadIdx.x;
    const bool v = i < d.n_events;
    const int32_t s = v ? d.session[i] : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, s);
    const int leader = __ffs(peers) - 1;
    int32_t at = 0;
    if (v && lane == leader) at = atomicAdd(&cursor[s], __popc(peers));
    at = __shfl_sync(0xffffffffu, at, leader);
    if (v) perm[off[s] + at + __popc(peers & lanemask_lt())] = (int32_t)i;
  }
}

// ---------------------------------------------------------------------------
// 4. sessions of <= 32 events: one warp each
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(OT) order_warp_kernel(const paste_order_desc d,
                                                        const int64_t* off, const int64_t* tbase,
                                                        const int32_t* perm, int32_t* nseg,
                                                        int32_t* big, OrderCounters* c) {
  __shared__ int32_t wseq[OT / 32][32];
  if (c->bad_session != 0) return;
  const bool grouped = c->ungrouped == 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n_warps = (int64_t)gridDim.x * (OT / 32);
  unsigned long long reord = 0;
  for (int64_t s = (int64_t)blockIdx.x * (OT / 32) + w; s < d.n_sessions; s += n_warps) {
    const int64_t o = off[s];
    const int64_t len64 = off[s + 1] - o;
    const int len = len64 > 64 ? 64 : (int)len64;
    if (len == 0) {
      if (lane == 0) nseg[s] = 0;
      continue;
    }
    if (len > 32) {
      if (lane == 0) big[atomicAdd(&c->n_big, 1ull)] = (int32_t)s;
      continue;
    }
    const bool v = lane < len;
    const int32_t idx = v ? (grouped ? (int32_t)(o + lane) : perm[o + lane]) : 0;
    OKey k = sentinel();
    int32_t sq = 0;
    if (v) {
      sq = d.seq[idx];
      k.t = norm_t(d.t_start[idx]);
      k.seq = sq;
      k.arr = idx;
    }
    // the arrival-order seq list (lane j: the seq of the j-th arrival)
    int arank = lane;
    if (!grouped) {
      arank = 0;
      for (int j = 0; j < len; ++j) arank += __shfl_sync(0xffffffffu, k.arr, j) < k.arr;
    }
    if (v) wseq[w][arank] = sq;
    __syncwarp();
    const int32_t aseq = wseq[w][lane];
    __syncwarp();
    // stable sort by (t_start, seq), only when the arrival order is not sorted
    const OKey nx = shfl_key(k, (lane + 1) & 31);
    const bool in_order = lane >= len - 1 || okey_less<1>(k, nx);
    if (!__all_sync(0xffffffffu, in_order)) {
#pragma unroll
      for (int k2 = 2; k2 <= 32; k2 <<= 1) {
#pragma unroll
        for (int j = k2 >> 1; j > 0; j >>= 1) {
          const OKey p = shfl_xor_key(k, j);
          const bool take_min = ((lane & j) == 0) == ((lane & k2) == 0);
          const bool pl = okey_less<1>(p, k);
          if (take_min ? pl : !pl) k = p;
        }
      }
    }
    const int32_t e = k.arr;
    if (__any_sync(0xffffffffu, v && k.seq != aseq) && lane == 0) ++reord;
    double ts = 0.0, te = 0.0;
    int32_t sig = -1;
    if (v) {
      ts = d.t_start[e];
      te = d.t_end[e];
      sig = d.sig[e];
    }
    const double pte = __shfl_up_sync(0xffffffffu, te, 1);
    const bool split = v && lane > 0 && ts - pte > d.inactivity_ms;
    const unsigned sb = __ballot_sync(0xffffffffu, split);
    const int lseg = __popc(sb & (lanemask_lt() | (1u << lane)));
    const bool tool = v && sig >= 0;
    const unsigned tb = __ballot_sync(0xffffffffu, tool);
    if (tool) {
      const int64_t p = tbase[s] + __popc(tb & lanemask_lt());
      d.out_session[p] = lseg;
      d.out_seq[p] = k.seq;
      d.out_t_start[p] = ts;
      d.out_t_end[p] = te;
      d.out_sig[p] = sig;
    }
    if (d.order && v) d.order[o + lane] = e;
    if (lane == 0) nseg[s] = 1 + __popc(sb);
  }
  if (reord) atomicAdd(&c->reordered, reord);
}

// ---------------------------------------------------------------------------
// 5. longer sessions: one CTA each
// ---------------------------------------------------------------------------
template <int MODE>
__device__ int merge_path(const OKey* a, int na, const OKey* b, int nb, int diag) {
  int lo = max(0, diag - nb), hi = min(diag, na);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (okey_less<MODE>(b[diag - 1 - mid], a[mid]))
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

// Sorts src[0, len) (global memory), using tmp as the ping-pong buffer;
// returns the buffer holding the result.  All threads of the CTA call it.
template <int MODE>
__device__ OKey* cta_sort(OKey* src, OKey* tmp, int len, OKey* sm) {
  for (int c0 = 0; c0 < len; c0 += CHUNK) {
    const int cl = min(CHUNK, len - c0);
    int P = 2;
    while (P < cl) P <<= 1;
    for (int j = threadIdx.x; j < P; j += CT) sm[j] = j < cl ? src[c0 + j] : sentinel();
    __syncthreads();
    for (int k2 = 2; k2 <= P; k2 <<= 1) {
      for (int j = k2 >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < P; i += CT) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const OKey a = sm[i], b = sm[ixj];
            const bool asc = (i & k2) == 0;
            if (asc ? okey_less<MODE>(b, a) : okey_less<MODE>(a, b)) {
              sm[i] = b;
              sm[ixj] = a;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int j = threadIdx.x; j < cl; j += CT) src[c0 + j] = sm[j];
    __syncthreads();
  }
  OKey* a = src;
  OKey* b = tmp;
  for (int wdt = CHUNK; wdt < len; wdt <<= 1) {
    for (int base = threadIdx.x * MIPT; base < len; base += CT * MIPT) {
      const int lo = base / (2 * wdt) * (2 * wdt);
      const int mid = min(lo + wdt, len), hi = min(lo + 2 * wdt, len);
      const OKey* x = a + lo;
      const OKey* y = a + mid;
      const int nx = mid - lo, ny = hi - mid;
      int i = merge_path<MODE>(x, nx, y, ny, base - lo);
      int j = base - lo - i;
      for (int q = 0; q < MIPT && base + q < hi; ++q) {
        const bool take_x = j >= ny || (i < nx && !okey_less<MODE>(y[j], x[i]));
        b[base + q] = take_x ? x[i++] : y[j++];
      }
    }
    __syncthreads();
    OKey* t = a;
    a = b;
    b = t;
  }
  return a;
}

__global__ void __launch_bounds__(CT) order_cta_kernel(const paste_order_desc d,
                                                       const int64_t* off, const int64_t* tbase,
                                                       const int32_t* perm, int32_t* nseg,
                                                       const int32_t* big, OKey* keyA, OKey* keyB,
                                                       int32_t* aseq_buf, OrderCounters* c) {
  __shared__ OKey sm[CHUNK];
  __shared__ int32_t wsum[2][CT / 32];
  __shared__ int flag;
  if (c->bad_session != 0) return;
  const bool grouped = c->ungrouped == 0;
  const int n_big = (int)c->n_big;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int b = blockIdx.x; b < n_big; b += gridDim.x) {
    const int64_t s = big[b];
    const int64_t o = off[s];
    const int len = (int)(off[s + 1] - o);
    OKey* A = keyA + o;
    OKey* B = keyB + o;
    int32_t* aseq = aseq_buf + o;
    for (int j = threadIdx.x; j < len; j += CT) {
      const int32_t idx = grouped ? (int32_t)(o + j) : perm[o + j];
      OKey k;
      k.t = norm_t(d.t_start[idx]);
      k.seq = d.seq[idx];
      k.arr = idx;
      A[j] = k;
    }
    __syncthreads();
    OKey* R = A;
    OKey* T = B;
    if (!grouped) {  // recover the arrival order first
      R = cta_sort<0>(A, B, len, sm);
      T = R == A ? B : A;
    }
    for (int j = threadIdx.x; j < len; j += CT) aseq[j] = R[j].seq;
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    int unsorted = 0;
    for (int j = threadIdx.x; j + 1 < len; j += CT) unsorted |= okey_less<1>(R[j + 1], R[j]);
    if (unsorted) flag = 1;
    __syncthreads();
    if (flag) R = cta_sort<1>(R, T, len, sm);
    // reorder check, gap split and tool ranks over the sorted session
    int seg_carry = 0, tool_carry = 0, reord = 0;
    for (int c0 = 0; c0 < len; c0 += CT) {
      const int j = c0 + threadIdx.x;
      const bool v = j < len;
      int32_t e = 0, sq = 0, sig = -1;
      double ts = 0.0, te = 0.0;
      bool split = false;
      if (v) {
        e = R[j].arr;
        sq = R[j].seq;
        ts = d.t_start[e];
        te = d.t_end[e];
        sig = d.sig[e];
        reord |= sq != aseq[j];
        if (j > 0) split = ts - d.t_end[R[j - 1].arr] > d.inactivity_ms;
      }
      const bool tool = v && sig >= 0;
      const unsigned sb = __ballot_sync(0xffffffffu, split);
      const unsigned tb = __ballot_sync(0xffffffffu, tool);
      if (lane == 0) {
        wsum[0][w] = __popc(sb);
        wsum[1][w] = __popc(tb);
      }
      __syncthreads();
      int sbase = seg_carry, tbase_w = tool_carry, stot = 0, ttot = 0;
      for (int q = 0; q < CT / 32; ++q) {
        if (q < w) {
          sbase += wsum[0][q];
          tbase_w += wsum[1][q];
        }
        stot += wsum[0][q];
        ttot += wsum[1][q];
      }
      __syncthreads();
      if (tool) {
        const int64_t p = tbase[s] + tbase_w + __popc(tb & lanemask_lt());
        d.out_session[p] = sbase + __popc(sb & (lanemask_lt() | (1u << lane)));
        d.out_seq[p] = sq;
        d.out_t_start[p] = ts;
        d.out_t_end[p] = te;
        d.out_sig[p] = sig;
      }
      if (d.order && v) d.order[o + j] = e;
      seg_carry += stot;
      tool_carry += ttot;
    }
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    if (reord) flag = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
      nseg[s] = 1 + seg_carry;
      if (flag) atomicAdd(&c->reordered, 1ull);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// 6. global segment numbers + results
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(OT) order_number_kernel(const paste_order_desc d,
                                                          const int64_t* tbase,
                                                          const int64_t* sbase,
                                                          const OrderCounters* c) {
  if (c->bad_session != 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t n_warps = (int64_t)gridDim.x * (OT / 32);
  for (int64_t s = (int64_t)blockIdx.x * (OT / 32) + (threadIdx.x >> 5); s < d.n_sessions;
       s += n_warps) {
    const int32_t add = (int32_t)sbase[s];
    for (int64_t p = tbase[s] + lane; p < tbase[s + 1]; p += 32) d.out_session[p] += add;
  }
}

__global__ void __launch_bounds__(OT) order_tok_kernel(const paste_order_desc d,
                                                       const int64_t* tbase,
                                                       const OrderCounters* c) {
  if (c->bad_session != 0) return;
  const int64_t n_out = tbase[d.n_sessions];
  for (int64_t p = (int64_t)blockIdx.x * OT + threadIdx.x; p < n_out;
       p += (int64_t)gridDim.x * OT) {
    const bool first = p == 0 || d.out_session[p] != d.out_session[p - 1];
    d.out_tok[p] = d.out_sig[p] | (first ? (int32_t)0x80000000 : 0);
  }
}

__global__ void order_finish_kernel(const paste_order_desc d, const int64_t* tbase,
                                    const int64_t* sbase, const OrderCounters* c) {
  const bool bad = c->bad_session != 0;
  *d.n_out = bad ? 0 : tbase[d.n_sessions];
  *d.n_segments = bad ? 0 : sbase[d.n_sessions];
  *d.reordered = bad ? 0 : (int64_t)c->reordered;
  *d.status = (c->nan_t ? PASTE_ORDER_NAN_T : 0) | (bad ? PASTE_ORDER_BAD_SESSION : 0);
}

struct OrderScratch {
  OrderCounters* counters;
  int32_t *cnt, *ntool, *nseg, *cursor, *big, *perm, *aseq;
  int64_t *off, *tbase, *sbase, *bsum;
  OKey *keyA, *keyB;
  int64_t bytes;
};

OrderScratch carve(char* base, int64_t n, int64_t S) {
  OrderScratch r{};
  int64_t at = 0;
  auto take = [&](int64_t b) {
    char* p = base ? base + at : nullptr;
    at += (b + 255) / 256 * 256;
    return p;
  };
  const int64_t nb = (S + SCAN_TILE - 1) / SCAN_TILE + 1;
  r.counters = reinterpret_cast<OrderCounters*>(take(sizeof(OrderCounters)));
  r.cnt = reinterpret_cast<int32_t*>(take(4 * S));
  r.ntool = reinterpret_cast<int32_t*>(take(4 * S));
  r.cursor = reinterpret_cast<int32_t*>(take(4 * S));
  r.nseg = reinterpret_cast<int32_t*>(take(4 * S));
  r.big = reinterpret_cast<int32_t*>(take(4 * S));
  r.off = reinterpret_cast<int64_t*>(take(8 * (S + 1)));
  r.tbase = reinterpret_cast<int64_t*>(take(8 * (S + 1)));
  r.sbase = reinterpret_cast<int64_t*>(take(8 * (S + 1)));
  r.bsum = reinterpret_cast<int64_t*>(take(8 * nb));
  r.perm = reinterpret_cast<int32_t*>(take(4 * n));
  r.aseq = reinterpret_cast<int32_t*>(take(4 * n));
  r.keyA = reinterpret_cast<OKey*>(take(sizeof(OKey) * n));
  r.keyB = reinterpret_cast<OKey*>(take(sizeof(OKey) * n));
  r.bytes = at;
  return r;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace
}  // namespace paste

extern "C" int64_t paste_ingest_order_scratch_bytes(int64_t n_events, int32_t n_sessions) {
  return paste::carve(nullptr, n_events < 0 ? 0 : n_events, n_sessions < 0 ? 0 : n_sessions).bytes;
}

extern "C" int paste_ingest_order(const paste_order_desc* d, void* scratch, int64_t scratch_bytes,
                                  void* stream) {
  using namespace paste;
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null order descriptor");
  PASTE_REQUIRE(d->n_events >= 0 && d->n_events < INT32_MAX, "n_events must be in [0, 2^31)");
  PASTE_REQUIRE(d->n_sessions >= 0, "n_sessions must be >= 0");
  PASTE_REQUIRE(d->n_out && d->n_segments && d->reordered && d->status, "null result pointer");
  PASTE_REQUIRE(d->n_events == 0 || (d->session && d->seq && d->t_start && d->t_end && d->sig &&
                                     d->out_session && d->out_seq && d->out_t_start &&
                                     d->out_t_end && d->out_sig),
                "null column");
  const int64_t n = d->n_events, S = d->n_sessions;
  OrderScratch sc = carve(static_cast<char*>(scratch), n, S);
  PASTE_REQUIRE(scratch != nullptr && scratch_bytes >= sc.bytes,
                "scratch too small: need %lld bytes", (long long)sc.bytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const paste_order_desc D = *d;
  // counters + the per-session counts / cursors (one contiguous memset)
  const int64_t zero_bytes = reinterpret_cast<char*>(sc.nseg) - reinterpret_cast<char*>(sc.counters);
  PASTE_CUDA_CHECK(cudaMemsetAsync(sc.counters, 0, (size_t)zero_bytes, st));
  const int grid_ev = (int)std::max<int64_t>(1, std::min<int64_t>((n + OT - 1) / OT,
                                                                  (int64_t)sm_count() * 8));
  const int grid_ss = (int)std::max<int64_t>(1, std::min<int64_t>((S + OT / 32 - 1) / (OT / 32),
                                                                  (int64_t)sm_count() * 16));
  int launches = 0;
  if (n > 0) {
    order_count_kernel<<<grid_ev, OT, 0, st>>>(D, sc.cnt, sc.ntool, sc.counters);
    ++launches;
  }
  int rc = scan_i32(sc.cnt, sc.off, S, sc.bsum, st);
  if (rc) return rc;
  rc = scan_i32(sc.ntool, sc.tbase, S, sc.bsum, st);
  if (rc) return rc;
  if (n > 0) {
    order_place_kernel<<<grid_ev, OT, 0, st>>>(D, sc.off, sc.cursor, sc.perm, sc.counters);
    ++launches;
  }
  if (S > 0) {
    order_warp_kernel<<<grid_ss, OT, 0, st>>>(D, sc.off, sc.tbase, sc.perm, sc.nseg, sc.big,
                                              sc.counters);
    order_cta_kernel<<<sm_count() * 2, CT, 0, st>>>(D, sc.off, sc.tbase, sc.perm, sc.nseg,
                                                    sc.big, sc.keyA, sc.keyB, sc.aseq,
                                                    sc.counters);
    launches += 2;
  }
  rc = scan_i32(sc.nseg, sc.sbase, S, sc.bsum, st);
  if (rc) return rc;
  if (S > 0) {
    order_number_kernel<<<grid_ss, OT, 0, st>>>(D, sc.tbase, sc.sbase, sc.counters);
    ++launches;
  }
  if (d->out_tok && n > 0) {
    order_tok_kernel<<<grid_ev, OT, 0, st>>>(D, sc.tbase, sc.counters);
    ++launches;
  }
  order_finish_kernel<<<1, 1, 0, st>>>(D, sc.tbase, sc.sbase, sc.counters);
  ++launches;
  count_launch(launches);
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
