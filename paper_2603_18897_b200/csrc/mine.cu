// K2 count_structural / K1 ingest / mining selection for sm_100a.
//
// Reference: mine() (mining.py:248-292) with its windows and distinct-
// subsequence support (mining.py:164-194, 266-275), anchored / contiguous
// matching (match_at, mining.py:119-156) and the per-context rescans of
// _collect_occurrences (mining.py:215-227).
//
// Reformulation (verified exact): every count mine()
// needs is a function of the (k+1)-grams of a session's tool tokens.  For
// position j of a stream s_0..s_{L-1}, T_j = (s_{j-k} .. s_{j-1}, s_j) with
// BEGIN before the stream:
//   * target j: window = the non-BEGIN part of (s_{j-k}..s_{j-1});
//     support[tool(s_j)][c] += 1 for each distinct subsequence c (anchored)
//     or suffix c (contiguous);
//   * anchor a = j-1 (s_{j-1} != BEGIN): the contexts that match at a are
//     u + (s_a) for each distinct subsequence u of the non-BEGIN part of
//     (s_{j-k}..s_{j-2}) (anchored, rightmost embedding is complete) or the
//     contiguous suffixes ending at a; follow[c][tool(s_j)] += 1.
//   * match[c] counts every anchor, including a segment's last event (no
//     target follows it): the anchors whose last k symbols are w number
//     sum_x H[(x, w)] -- a marginal of the same histogram, so no END grams
//     are counted.
// So the device counts one histogram H over (k+1)-grams (one increment per
// event) and expands it once.
//
// Token stream format: int32 sig ids with bit 31 set on the first token of
// every segment (session after gap splitting).
#include "common.cuh"

#include <cooperative_groups.h>
#include <mutex>
#include <unordered_map>

namespace paste {

constexpr uint32_t SEG_START = 0x80000000u;
constexpr int MT = 256;  // threads per CTA

struct MineGeom {
  int S;      // signatures
  int T;      // tools (S / 2)
  int k;
  int base;   // S + 2 (BEGIN = S, END = S + 1)
  int64_t n_bins;
  int64_t n_ctx;      // sum_{n=1..k} S^n
  int64_t ctx_off[17];  // start of length-n contexts
  int64_t pw[18];       // S^i
};

__device__ __forceinline__ int64_t ctx_index(const MineGeom& g, const int* c, int n) {
  int64_t idx = 0;
  for (int i = 0; i < n; ++i) idx = idx * g.S + c[i];
  return g.ctx_off[n] + idx;
}

// ---------------------------------------------------------------------------
// count: one (k+1)-gram per token
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(MT) count_grams_kernel(const uint32_t* __restrict__ tok,
                                                         int64_t n, MineGeom g,
                                                         uint32_t* __restrict__ hist) {
  const int64_t i = (int64_t)blockIdx.x * MT + threadIdx.x;
  const unsigned lanes = __ballot_sync(0xffffffffu, i < n);
  if (i >= n) return;
  const uint32_t t = __ldg(tok + i);
  // gram ending at i: walk back until a segment start
  int64_t key = (int64_t)(t & ~SEG_START);
  int64_t mult = g.base;
  bool stop = (t & SEG_START) != 0;
  for (int d = 1; d <= g.k; ++d) {
    int sym = g.S;  // BEGIN
    if (!stop) {
      const uint32_t p = __ldg(tok + i - d);
      sym = (int)(p & ~SEG_START);
      stop = (p & SEG_START) != 0;
    }
    key += (int64_t)sym * mult;
    mult *= g.base;
  }
  // warp-aggregated increment (skewed traces repeat grams within a warp)
  const unsigned peers = __match_any_sync(lanes, key);
  if ((__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(hist + key, (uint32_t)__popc(peers));
}

// ---------------------------------------------------------------------------
// expand: (k+1)-gram histogram -> tool_count / support / match / follow
//
// One warp per *window* w = (s_k .. s_1) (the k symbols before the target),
// lanes over the target symbol s_0: the histogram row H[w][*] is contiguous
// (key = s_0 + base * w), so a warp reads it with one coalesced load and every
// table update of the window is aggregated across lanes first:
//   * support[t][c] += sum_{s_0 in tool t} H   for each distinct subsequence c
//     of the window (or suffix, contiguous relation);
//   * match[c]      += sum_{all s_0} H        for each context c matching at
//     the anchor s_1 (distinct subsequence of (s_k..s_2) + s_1);
//   * follow[c][t]  += sum_{s_0 in tool t} H   for the same contexts.
// Distinct subsequences are enumerated as index masks and kept only in their
// leftmost embedding (each chosen position is the first occurrence of its
// symbol after the previous chosen one), which lists each distinct
// subsequence exactly once without comparing masks.  Length-1 contexts and
// tool_count (hit by every window) accumulate in shared memory per CTA.
// ---------------------------------------------------------------------------
constexpr int XT = 256;                 // threads per expand CTA
constexpr int XSMEM_CELLS = 4096;       // u64 cells for the length-1 / tool caches

template <int K>
__device__ __forceinline__ int window_contexts(const MineGeom& g, const int* w, int wl, bool anchored,
                                               bool with_empty, int tail, int64_t* out) {
  // contexts = (distinct subsequence | suffix of w[0..wl)) + (tail if >= 0)
  int n = 0;
  if (anchored) {
#pragma unroll
    for (int mask = 0; mask < (1 << K); ++mask) {
      if ((mask >> wl) != 0 || (mask == 0 && !with_empty)) continue;
      bool canon = true;
      int prev = -1, len = 0;
      int64_t v = 0;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (i < wl && ((mask >> i) & 1)) {
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (q > prev && q < i && !((mask >> q) & 1) && w[q] == w[i]) canon = false;
          prev = i;
          v = v * g.S + w[i];
          ++len;
        }
      }
      if (!canon) continue;
      if (tail >= 0) {
        v = v * g.S + tail;
        ++len;
      }
      out[n++] = g.ctx_off[len] + v;
    }
  } else {
#pragma unroll
    for (int st = 0; st <= K; ++st) {
      if (st > wl || (st == wl && !with_empty)) continue;
      int64_t v = 0;
      int len = 0;
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i >= st && i < wl) {
          v = v * g.S + w[i];
          ++len;
        }
      if (tail >= 0) {
        v = v * g.S + tail;
        ++len;
      }
      out[n++] = g.ctx_off[len] + v;
    }
  }
  return n;
}

// 64-bit add into a (lo, hi) pair of shared u32 counters with native 32-bit
// atomics (a shared u64 atomicAdd compiles to a CAS loop)
__device__ __forceinline__ void smem_add64(uint32_t* cell, unsigned long long v) {
  const uint32_t lo = (uint32_t)v;
  uint32_t hi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(cell, lo);
  hi += (uint32_t)(old + lo < old);  // carry
  if (hi) atomicAdd(cell + 1, hi);
}

template <int K>
__global__ void __launch_bounds__(XT) expand_windows_kernel(
    const uint32_t* __restrict__ hist, MineGeom g, int relation, unsigned long long* tool_count,
    unsigned long long* support, unsigned long long* match, unsigned long long* follow,
    int use_cache) {
  // cache (u64 as lo/hi u32 pairs): tool_count[T] | support[T][S] (length-1)
  // | match[S] | follow[S][T]
  __shared__ uint32_t cache[2 * XSMEM_CELLS];
  const int S = g.S, T = g.T, base = g.base, BEGIN = S, END = S + 1;
  uint32_t* c_tool = cache;
  uint32_t* c_sup = cache + 2 * T;
  uint32_t* c_match = c_sup + 2 * (int64_t)T * S;
  uint32_t* c_follow = c_match + 2 * S;
  const int cells = T + 2 * T * S + S;
  if (use_cache)
    for (int i = threadIdx.x; i < 2 * cells; i += XT) cache[i] = 0;
  __syncthreads();
  const bool anchored = relation == PASTE_REL_ANCHORED;
  const int lane = threadIdx.x & 31;
  const int64_t n_win = g.n_bins / base;
  const int64_t pw_k = n_win;  // base^K
  const int64_t warp0 = ((int64_t)blockIdx.x * XT + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * XT) >> 5;
  for (int64_t wi = warp0; wi < n_win; wi += n_warps) {
    // decode the window, oldest first; BEGINs must be a prefix, no END
    int sym[K + 1];
    {
      uint32_t v = (uint32_t)wi;  // n_win < 2^31 (geometry check)
#pragma unroll
      for (int d = 1; d <= K; ++d) {
        sym[d] = (int)(v % (uint32_t)base);
        v /= (uint32_t)base;
      }
    }
    int nb = 0;
    bool valid = true;
#pragma unroll
    for (int d = K; d >= 1; --d) {
      if (sym[d] == END) valid = false;
      if (sym[d] == BEGIN) {
        if (nb != K - d) valid = false;
        ++nb;
      }
    }
    if (!valid) continue;  // never counted (an all-BEGIN window still counts tool_count)
    const uint32_t* row = hist + wi * base;
    int win[K];
    const int wl = K - nb;
#pragma unroll
    for (int i = 0; i < K; ++i) win[i] = i < wl ? sym[wl - i] : 0;
    // contexts of this window (warp-uniform)
    int64_t sup_ctx[(1 << K)];
    int64_t mt_ctx[(1 << K)];
    const int n_sup = wl > 0 ? window_contexts<K>(g, win, wl, anchored, false, -1, sup_ctx) : 0;
    const bool has_anchor = wl > 0;  // s_1 is a real event
    const int n_mt =
        has_anchor ? window_contexts<K>(g, win, wl - 1, anchored, true, sym[1], mt_ctx) : 0;
    // anchors whose last K symbols are this window: sum over the symbol
    // before it (hist[x * base^K + wi], all x)
    unsigned long long tot = 0;
    if (n_mt > 0)
      for (int x = lane; x < base; x += 32) tot += __ldg(hist + (int64_t)x * pw_k + wi);
    for (int c0 = 0; c0 < base; c0 += 32) {
      const int s0 = c0 + lane;
      const uint32_t h = s0 < base ? __ldg(row + s0) : 0u;
      if (__ballot_sync(0xffffffffu, h != 0) == 0) continue;
      // per-tool sums in the even lane of each (2t, 2t+1) pair
      const unsigned long long hs = s0 < S ? h : 0u;
      const unsigned long long ht = hs + __shfl_xor_sync(0xffffffffu, hs, 1);
      if ((s0 & 1) || ht == 0) continue;
      const int t = s0 >> 1;
      if (use_cache) smem_add64(c_tool + 2 * t, ht);
      else atomicAdd(tool_count + t, ht);
#pragma unroll
      for (int q = 0; q < (1 << K); ++q) {
        if (q >= n_sup) break;
        const int64_t c = sup_ctx[q];
        if (use_cache && c < S) smem_add64(c_sup + 2 * ((int64_t)t * S + c), ht);
        else atomicAdd(support + (int64_t)t * g.n_ctx + c, ht);
      }
#pragma unroll
      for (int q = 0; q < (1 << K); ++q) {
        if (q >= n_mt) break;
        const int64_t c = mt_ctx[q];
        if (use_cache && c < S) smem_add64(c_follow + 2 * (c * T + t), ht);
        else atomicAdd(follow + c * T + t, ht);
      }
    }
    if (n_mt == 0) continue;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (tot == 0) continue;
    if (lane < n_mt) {
      int64_t c = 0;
#pragma unroll
      for (int q = 0; q < (1 << K); ++q)
        if (q == lane) c = mt_ctx[q];
      if (use_cache && c < S) smem_add64(c_match + 2 * c, tot);
      else atomicAdd(match + c, tot);
    }
  }
  if (!use_cache) return;
  __syncthreads();
  for (int i = threadIdx.x; i < cells; i += XT) {
    const unsigned long long v =
        (unsigned long long)cache[2 * i] | ((unsigned long long)cache[2 * i + 1] << 32);
    if (v == 0) continue;
    if (i < T) {
      atomicAdd(tool_count + i, v);
    } else if (i < T + T * S) {
      const int j = i - T, t = j / S, c = j - t * S;
      atomicAdd(support + (int64_t)t * g.n_ctx + c, v);
    } else if (i < T + T * S + S) {
      atomicAdd(match + (i - T - T * S), v);
    } else {
      atomicAdd(follow + (i - T - T * S - S), v);  // follow[c][t], c < S
    }
  }
}

// ---------------------------------------------------------------------------
// target-sliced tail: the same expansion over one block of histogram columns
// (s0 in [lo, lo + W)), read from the s0-major slice [s0 - lo][window].
// Windows with no count in the block and an anchor outside it are skipped
// before their contexts are enumerated.
// ---------------------------------------------------------------------------
__global__ void transpose_slices_kernel(const uint32_t* __restrict__ hist, int64_t n_win, int base,
                                        int S, int cols, uint32_t* __restrict__ out) {
  // out[c][w] = hist[w * base + c] (c < S), 0 for S <= c < cols
  const int64_t total = (int64_t)cols * n_win;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / n_win, w = i - c * n_win;
    out[i] = c < S ? __ldg(hist + w * base + c) : 0u;
  }
}

template <int K>
__global__ void __launch_bounds__(XT) expand_slice_kernel(
    const uint32_t* __restrict__ slice, int lo, int width, MineGeom g, int relation,
    unsigned long long* tool_count, unsigned long long* support, unsigned long long* match,
    unsigned long long* follow) {
  const int S = g.S, T = g.T, base = g.base, BEGIN = S, END = S + 1;
  const bool anchored = relation == PASTE_REL_ANCHORED;
  const int lane = threadIdx.x & 31;
  const int64_t n_win = g.n_bins / base;
  const int64_t warp0 = ((int64_t)blockIdx.x * XT + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * XT) >> 5;
  for (int64_t wi = warp0; wi < n_win; wi += n_warps) {
    int sym[K + 1];
    {
      uint32_t v = (uint32_t)wi;
#pragma unroll
      for (int d = 1; d <= K; ++d) {
        sym[d] = (int)(v % (uint32_t)base);
        v /= (uint32_t)base;
      }
    }
    int nb = 0;
    bool valid = true;
#pragma unroll
    for (int d = K; d >= 1; --d) {
      if (sym[d] == END) valid = false;
      if (sym[d] == BEGIN) {
        if (nb != K - d) valid = false;
        ++nb;
      }
    }
    if (!valid) continue;
    const int wl = K - nb;
    const bool anchor_here = wl > 0 && sym[1] >= lo && sym[1] < lo + width;
    // this block's counts of the window (lane = column - lo, width <= 32 per chunk)
    bool any = false;
    for (int c0 = 0; c0 < width && !any; c0 += 32)
      any = __ballot_sync(0xffffffffu, c0 + lane < width &&
                                           __ldg(slice + (int64_t)(c0 + lane) * n_win + wi) != 0u) != 0;
    if (!any && !anchor_here) continue;
    int win[K];
#pragma unroll
    for (int i = 0; i < K; ++i) win[i] = i < wl ? sym[wl - i] : 0;
    int64_t sup_ctx[(1 << K)];
    int64_t mt_ctx[(1 << K)];
    const int n_sup = wl > 0 ? window_contexts<K>(g, win, wl, anchored, false, -1, sup_ctx) : 0;
    const int n_mt = wl > 0 ? window_contexts<K>(g, win, wl - 1, anchored, true, sym[1], mt_ctx) : 0;
    for (int c0 = 0; c0 < width; c0 += 32) {
      const int col = c0 + lane;
      const uint32_t h = col < width ? __ldg(slice + (int64_t)col * n_win + wi) : 0u;
      if (__ballot_sync(0xffffffffu, h != 0) == 0) continue;
      const int s0 = lo + col;  // lo and width are even: tool pairs share a chunk
      const unsigned long long hs = s0 < S ? h : 0u;
      const unsigned long long ht = hs + __shfl_xor_sync(0xffffffffu, hs, 1);
      if ((s0 & 1) || ht == 0) continue;
      const int t = s0 >> 1;
      atomicAdd(tool_count + t, ht);
#pragma unroll
      for (int q = 0; q < (1 << K); ++q) {
        if (q >= n_sup) break;
        atomicAdd(support + (int64_t)t * g.n_ctx + sup_ctx[q], ht);
      }
#pragma unroll
      for (int q = 0; q < (1 << K); ++q) {
        if (q >= n_mt) break;
        atomicAdd(follow + mt_ctx[q] * T + t, ht);
      }
    }
    if (!anchor_here || n_mt == 0) continue;
    // anchors whose last K symbols are this window: the grams x*base^K + wi,
    // all of column sym[1] (row x*base^(K-1) + wi/base of the s0-major slice)
    const int64_t pw1 = n_win / base;  // base^(K-1)
    const uint32_t* col = slice + (int64_t)(sym[1] - lo) * n_win + wi / base;
    unsigned long long tot = 0;
    for (int x = lane; x < base; x += 32) tot += __ldg(col + (int64_t)x * pw1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (tot == 0) continue;
    if (lane < n_mt) {
      int64_t c = 0;
#pragma unroll
      for (int q = 0; q < (1 << K); ++q)
        if (q == lane) c = mt_ctx[q];
      atomicAdd(match + c, tot);
    }
  }
}

// ---------------------------------------------------------------------------
// select: (target, context) pairs clearing the sigma gates and the tau bound
// ---------------------------------------------------------------------------
__global__ void select_kernel(MineGeom g, const unsigned long long* tool_count,
                              const unsigned long long* support, const unsigned long long* match,
                              const unsigned long long* follow, int64_t sigma, double tau,
                              int64_t cap, unsigned long long* n_out, int64_t* out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)g.T * g.n_ctx) return;
  const int t = (int)(idx / g.n_ctx);
  const int64_t c = idx - (int64_t)t * g.n_ctx;
  const unsigned long long sup = support[idx];
  if (sup < (unsigned long long)sigma || tool_count[t] < (unsigned long long)sigma) return;
  const unsigned long long mt = match[c];
  if (mt == 0) return;  // mining.py:278
  const unsigned long long fl = follow[c * g.T + t];
  // p <= follow / match for any mapping (hits <= len(occ)); below tau it can never pass
  if (__ddiv_rn((double)fl, (double)mt) < tau) return;
  const unsigned long long slot = atomicAdd(n_out, 1ull);
  if ((int64_t)slot >= cap) return;
  int64_t* o = out + 5 * slot;
  o[0] = t;
  o[1] = c;
  o[2] = (int64_t)sup;
  o[3] = (int64_t)mt;
  o[4] = (int64_t)fl;
}

// ---------------------------------------------------------------------------
// sorted selection for mapping-free mining (columnar traces): the candidates
// that clear sigma and p = follow / match >= tau, in mine()'s output order
// (_sort_key, mining.py:105-111): -p, -len(context), target name, context.
// Sig / tool ids are interned in sorted name order, so with
//   hi = ~bits(p)                       (p > 0: bit order == numeric order)
//   lo = (k - len) << 60 | tool << 40 | base-S digits of the context
// the order is (hi, lo) ascending and every key is distinct ((t, c) unique).
// The sort is a rank count: rank[i] = #{j : key_j < key_i} over tiles of keys
// staged in shared memory (persistent CTAs over (i-tile, j-tile) pairs), then
// a scatter.
// ---------------------------------------------------------------------------
struct SelRow {
  int64_t tool, ctx, support, match, follow;
  double p;
};

__global__ void select_keyed_kernel(MineGeom g, const unsigned long long* tool_count,
                                    const unsigned long long* support,
                                    const unsigned long long* match,
                                    const unsigned long long* follow, int64_t sigma, double tau,
                                    int64_t cap, unsigned long long* n_out, SelRow* rows,
                                    ulonglong2* keys) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)g.T * g.n_ctx) return;
  const int t = (int)(idx / g.n_ctx);
  const int64_t c = idx - (int64_t)t * g.n_ctx;
  const unsigned long long sup = support[idx];
  if (sup < (unsigned long long)sigma || tool_count[t] < (unsigned long long)sigma) return;
  const unsigned long long mt = match[c];
  if (mt == 0) return;
  const unsigned long long fl = follow[c * g.T + t];
  const double p = __ddiv_rn((double)fl, (double)mt);  // == Python's int / int
  if (p < tau) return;
  const unsigned long long slot = atomicAdd(n_out, 1ull);
  if ((int64_t)slot >= cap) return;
  int len = 1;
  while (len < g.k && c >= g.ctx_off[len + 1]) ++len;
  rows[slot] = SelRow{t, c, (int64_t)sup, (int64_t)mt, (int64_t)fl, p};
  keys[slot] = make_ulonglong2(~(unsigned long long)__double_as_longlong(p),
                               ((unsigned long long)(g.k - len) << 60) |
                                   ((unsigned long long)t << 40) |
                                   (unsigned long long)(c - g.ctx_off[len]));
}

constexpr int RI = 256, RJ = 128;

__global__ void __launch_bounds__(RI) rank_keys_kernel(const ulonglong2* __restrict__ keys,
                                                       const unsigned long long* n_out,
                                                       int64_t cap, uint32_t* rank) {
  __shared__ ulonglong2 tile[RJ];
  const unsigned long long nn = *n_out;
  const int64_t n = (int64_t)nn < cap ? (int64_t)nn : cap;
  const int64_t ni = (n + RI - 1) / RI, nj = (n + RJ - 1) / RJ;
  for (int64_t item = blockIdx.x; item < ni * nj; item += gridDim.x) {
    const int64_t it = item / nj, jt = item - it * nj;
    const int64_t j0 = jt * RJ;
    const int jn = (int)(n - j0 < RJ ? n - j0 : RJ);
    __syncthreads();
    for (int j = threadIdx.x; j < jn; j += RI) tile[j] = keys[j0 + j];
    __syncthreads();
    const int64_t i = it * RI + threadIdx.x;
    if (i >= n) continue;
    const ulonglong2 me = keys[i];
    uint32_t cnt = 0;
    for (int j = 0; j < jn; ++j) {
      const ulonglong2 o = tile[j];
      cnt += (o.x < me.x) | ((o.x == me.x) & (o.y < me.y));
    }
    if (cnt) atomicAdd(rank + i, cnt);
  }
}

__global__ void scatter_rows_kernel(const SelRow* __restrict__ rows, const uint32_t* __restrict__ rank,
                                    const unsigned long long* n_out, int64_t cap, SelRow* out) {
  const unsigned long long nn = *n_out;
  const int64_t n = (int64_t)nn < cap ? (int64_t)nn : cap;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[rank[i]] = rows[i];
}

static int make_geom(int n_sigs, int k, MineGeom* g) {
  if (n_sigs < 1 || k < 1 || k > 6 || n_sigs > (1 << 20)) return -1;
  g->S = n_sigs;
  g->T = (n_sigs + 1) / 2;
  g->k = k;
  g->base = n_sigs + 2;
  g->pw[0] = 1;
  for (int i = 1; i <= k + 1; ++i) {
    g->pw[i] = g->pw[i - 1] * n_sigs;
    if (g->pw[i] > ((int64_t)1 << 40)) return -1;
  }
  g->ctx_off[0] = 0;
  g->ctx_off[1] = 0;
  for (int n = 1; n <= k; ++n) g->ctx_off[n + 1] = g->ctx_off[n] + g->pw[n];
  g->n_ctx = g->ctx_off[k + 1];
  int64_t bins = 1;
  for (int i = 0; i <= k; ++i) {
    bins *= g->base;
    if (bins > ((int64_t)1 << 31)) return -1;
  }
  g->n_bins = bins;
  return 0;
}

}  // namespace paste

using namespace paste;

static inline unsigned long long* U64(uint64_t* p) { return reinterpret_cast<unsigned long long*>(p); }

extern "C" int paste_mine_geometry(int32_t n_sigs, int32_t k, int64_t* n_bins, int64_t* n_ctx) {
  MineGeom g;
  if (make_geom(n_sigs, k, &g) != 0) {
    set_error("mining geometry out of range (n_sigs=%d, k=%d)", n_sigs, k);
    return PASTE_ERR_UNSUPPORTED;
  }
  *n_bins = g.n_bins;
  *n_ctx = g.n_ctx;
  return PASTE_OK;
}

extern "C" int paste_mine_count(const paste_mine_desc* d, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null descriptor");
  MineGeom g;
  if (make_geom(d->n_sigs, d->k, &g) != 0) {
    set_error("mining geometry out of range (n_sigs=%d, k=%d)", d->n_sigs, d->k);
    return PASTE_ERR_UNSUPPORTED;
  }
  if (d->n_tokens > 0) {
    const int64_t blocks = (d->n_tokens + MT - 1) / MT;
    count_grams_kernel<<<(unsigned)blocks, MT, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const uint32_t*>(d->tokens), d->n_tokens, g, d->hist);
    count_launch();
    PASTE_CUDA_CHECK(cudaGetLastError());
  }
  return PASTE_OK;
}

extern "C" int paste_mine_expand(const paste_mine_desc* d, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null descriptor");
  MineGeom g;
  if (make_geom(d->n_sigs, d->k, &g) != 0) {
    set_error("mining geometry out of range (n_sigs=%d, k=%d)", d->n_sigs, d->k);
    return PASTE_ERR_UNSUPPORTED;
  }
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t n_win = g.n_bins / g.base;
  const int64_t want = (n_win + XT / 32 - 1) / (XT / 32);
  const int64_t cap = (int64_t)sms * 3;
  const unsigned grid = (unsigned)(want < cap ? (want > 0 ? want : 1) : cap);
  const int use_cache = (int64_t)g.T + 2 * (int64_t)g.T * g.S + g.S <= XSMEM_CELLS;
  int rc = -1;
#define PASTE_EXPAND(KV)                                                                     \
  if (d->k == KV) {                                                                          \
    expand_windows_kernel<KV><<<grid, XT, 0, (cudaStream_t)stream>>>(                        \
        d->hist, g, d->relation, U64(d->tool_count), U64(d->support), U64(d->match),         \
        U64(d->follow), use_cache);                                                          \
    rc = 0;                                                                                  \
  }
  PASTE_EXPAND(1) PASTE_EXPAND(2) PASTE_EXPAND(3) PASTE_EXPAND(4) PASTE_EXPAND(5) PASTE_EXPAND(6)
#undef PASTE_EXPAND
  PASTE_REQUIRE(rc == 0, "k=%d outside the expand kernel's range", d->k);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

extern "C" int32_t paste_mine_slice_cols(int32_t n_sigs, int32_t n_slices) {
  if (n_sigs < 1 || n_slices < 1) return 0;
  const int32_t tools = (n_sigs + 1) / 2;
  return 2 * ((tools + n_slices - 1) / n_slices);
}

extern "C" int paste_mine_transpose_slices(const paste_mine_desc* d, int32_t n_slices,
                                           uint32_t* hist_t, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr && hist_t != nullptr && d->hist != nullptr, "null argument");
  MineGeom g;
  if (make_geom(d->n_sigs, d->k, &g) != 0) {
    set_error("mining geometry out of range (n_sigs=%d, k=%d)", d->n_sigs, d->k);
    return PASTE_ERR_UNSUPPORTED;
  }
  const int32_t w = paste_mine_slice_cols(d->n_sigs, n_slices);
  PASTE_REQUIRE(w > 0, "n_slices must be >= 1");
  const int64_t n_win = g.n_bins / g.base;
  const int64_t total = (int64_t)w * n_slices * n_win;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  transpose_slices_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      d->hist, n_win, g.base, g.S, w * n_slices, hist_t);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

extern "C" int paste_mine_expand_slice(const paste_mine_desc* d, const uint32_t* slice,
                                       int32_t col_lo, int32_t slice_cols, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr && slice != nullptr, "null argument");
  PASTE_REQUIRE(col_lo >= 0 && slice_cols > 0 && (col_lo % 2) == 0 && (slice_cols % 2) == 0,
                "slice columns must be a non-empty even-aligned block");
  MineGeom g;
  if (make_geom(d->n_sigs, d->k, &g) != 0) {
    set_error("mining geometry out of range (n_sigs=%d, k=%d)", d->n_sigs, d->k);
    return PASTE_ERR_UNSUPPORTED;
  }
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t n_win = g.n_bins / g.base;
  // one warp per window: the per-window work is a short dependent chain
  // (block counts -> contexts -> atomics), so latency hiding wants every
  // window in flight at once
  const int64_t want = (n_win + XT / 32 - 1) / (XT / 32);
  const unsigned grid = (unsigned)(want > 0 ? want : 1);
  (void)sms;
  int rc = -1;
#define PASTE_EXPAND_SLICE(KV)                                                               \
  if (d->k == KV) {                                                                          \
    expand_slice_kernel<KV><<<grid, XT, 0, (cudaStream_t)stream>>>(                          \
        slice, col_lo, slice_cols, g, d->relation, U64(d->tool_count), U64(d->support),      \
        U64(d->match), U64(d->follow));                                                      \
    rc = 0;                                                                                  \
  }
  PASTE_EXPAND_SLICE(1) PASTE_EXPAND_SLICE(2) PASTE_EXPAND_SLICE(3) PASTE_EXPAND_SLICE(4)
  PASTE_EXPAND_SLICE(5) PASTE_EXPAND_SLICE(6)
#undef PASTE_EXPAND_SLICE
  PASTE_REQUIRE(rc == 0, "k=%d outside the expand kernel's range", d->k);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

extern "C" int paste_mine_select(const paste_mine_desc* d, int64_t sigma, double tau, int64_t cap,
                                 uint64_t* n_out, int64_t* out, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr && n_out != nullptr && out != nullptr, "null argument");
  MineGeom g;
  if (make_geom(d->n_sigs, d->k, &g) != 0) {
    set_error("mining geometry out of range (n_sigs=%d, k=%d)", d->n_sigs, d->k);
    return PASTE_ERR_UNSUPPORTED;
  }
  const int64_t total = (int64_t)g.T * g.n_ctx;
  const int threads = 256;
  select_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
      g, U64(d->tool_count), U64(d->support), U64(d->match), U64(d->follow), sigma, tau, cap,
      reinterpret_cast<unsigned long long*>(n_out), out);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

// ---------------------------------------------------------------------------
// K1 + K2 fused: columnar trace events -> segments -> (k+1)-gram histogram.
//
// Ingest semantics (ingest_trace / _split_on_gaps, events.py:196-252) for a
// columnar trace whose events are already grouped by session in first-
// appearance order and sorted by (t_start, seq) inside a session: a new
// segment starts at event y when y opens a session or
// t_start[y] - t_end[y-1] > inactivity (fp64, strict).  Order violations are
// counted (the host rejects unsorted input).  Each CTA stages a tile of
// events plus a (k+1)-event halo in shared memory with coalesced loads.
// ---------------------------------------------------------------------------
// Pipeline: one producer warp streams tiles of CTILE events (five columns,
// TMA bulk copies) into CNST shared-memory stages guarded by full / empty
// mbarriers.  Tiles are handed out dynamically (a global tile counter the
// producer bumps), so SMs that see slower L2 atomics do not set the tail.
// Each of the CW consumer warps owns 64 consecutive events of a tile (two
// 32-lane sub-chunks): segment flags come from the staged columns, the
// (k+1)-gram window from warp shuffles over the two sub-chunks plus one halo
// word per lane (the k events before the span, and the event after it), so
// consumers never wait on each other: no __syncthreads in the steady state.
//
// Counting: the grams of a segment's first two events, (BEGIN.., s_1, s_0),
// are shared by every segment (1/4 of all increments at a mean length of 8)
// and would serialise on a few L2 atomic units; they accumulate in a dense
// per-CTA shared-memory table of base^2 counters flushed once.  Every other
// gram is spread over ~1M bins and goes straight to L2 as a RED.
constexpr int CW = 8;                   // consumer warps
constexpr int CT = 32 * (CW + 1);       // + one producer warp
constexpr int CTILE = 64 * CW;          // events per tile (64 per consumer warp)
constexpr int CPRE = 8;                 // halo before the tile (>= k + 1, 16-B aligned)
constexpr int CSPAN = CTILE + 16;       // staged events per tile (halo + 1 after, padded)
constexpr int CNST = 4;                 // pipeline stages
constexpr int CHOT_MAX = 2048;          // dense hot-gram table capacity (u32)

// one stage of staged columns
struct __align__(16) ColumnTile {
  double ts[CSPAN];
  double te[CSPAN];
  int32_t sess[CSPAN];
  int32_t seq[CSPAN];
  int32_t sig[CSPAN];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Producer warp: fill stage T with tile t.  The 16-byte-granular part goes by
// bulk copy; the last < 4 events of the trace (arrays need not be padded) are
// stored by the lanes before lane 0's arrive releases them with the copy.
__device__ __forceinline__ void produce_tile(const paste_columnar_desc& C, int64_t t, ColumnTile* T,
                                             uint64_t* full, int lane) {
  const int64_t n = C.n_events;
  const int64_t g0 = t * CTILE - CPRE;
  const int64_t lo = g0 < 0 ? 0 : g0;
  int64_t hi = g0 + CSPAN;
  if (hi > n) hi = n;
  const int64_t cnt = (hi - lo) & ~(int64_t)3;
  for (int64_t x = lo + cnt + lane; x < hi; x += 32) {
    const int l = (int)(x - g0);
    T->ts[l] = C.t_start[x];
    T->te[l] = C.t_end[x];
    T->sess[l] = C.session[x];
    T->seq[l] = C.seq[x];
    T->sig[l] = C.sig[x];
  }
  __syncwarp();
  if (lane == 0) {
    const int off = (int)(lo - g0);
    const uint32_t b4 = (uint32_t)cnt * 4, b8 = (uint32_t)cnt * 8;
    mbar_expect_tx(full, cnt > 0 ? 3 * b4 + 2 * b8 : 0);
    if (cnt > 0) {
      bulk_g2s(T->ts + off, C.t_start + lo, b8, full);
      bulk_g2s(T->te + off, C.t_end + lo, b8, full);
      bulk_g2s(T->sess + off, C.session + lo, b4, full);
      bulk_g2s(T->seq + off, C.seq + lo, b4, full);
      bulk_g2s(T->sig + off, C.sig + lo, b4, full);
    }
  }
}

// v(l) = sig | segment-start flag << 31 for staged slot l (event x = g0 + l).
// Events before the trace start or past its end read as segment starts.
__device__ __forceinline__ uint32_t slot_word(const ColumnTile* T, int l, int64_t x, int64_t n,
                                              double gap) {
  if (x <= 0 || x >= n) return (x == 0 ? (uint32_t)T->sig[l] : 0u) | SEG_START;
  const bool b = (T->sess[l] != T->sess[l - 1]) || (__dsub_rn(T->ts[l], T->te[l - 1]) > gap);
  return (uint32_t)T->sig[l] | (b ? SEG_START : 0u);
}
// Count the gram ending at an event (window words w[1..K], w[0] = own
// word).  Hot grams go to the CTA's shared table.  Cold grams go straight to
// L2 (STAGE = false), or are returned as a staged word for
// stage_hist_kernel (STAGE = true): the gram key, bit 31 = already counted.
//
// Success lattice: a gram whose K+1 events are all successful (odd
// signatures, no BEGIN) is staged as STG_LAT | its index over the (S/2)^(K+1)
// lattice, which stage_hist_kernel counts in shared memory.  With the usual
// few-percent failure rate these are most full-window grams.
constexpr uint32_t STG_HOT = 0x80000000u, STG_KEY = 0x7fffffffu, STG_LAT = 0x40000000u;
constexpr uint32_t LAT_MAX = 65536;  // lattice cells (16-bit counters, 128 KB)
constexpr int STG_REPS = 8;  // histogram replicas of the L2 pass
__host__ __device__ inline int64_t stage_words(int64_t n) { return (n + 3) & ~(int64_t)3; }

template <int K, bool STAGE>
__device__ __forceinline__ uint32_t count_event(const uint32_t (&w)[K + 1], uint32_t S,
                                                uint32_t base, uint32_t hot_lo, uint32_t hot_n,
                                                uint32_t* hot, uint32_t* hist, uint32_t lat_t) {
  const uint32_t s0 = w[0] & 0x7fffffffu;
  uint32_t key = s0, mult = base;
  uint32_t li = s0 >> 1, lm = lat_t;  // success-lattice index (base lat_t digits)
  bool lat = STAGE && lat_t != 0 && (s0 & 1u);
  bool stop = w[0] >> 31;
#pragma unroll
  for (int d = 1; d <= K; ++d) {
    const uint32_t sd = w[d] & 0x7fffffffu;
    key += (stop ? S : sd) * mult;
    lat = lat && !stop && (sd & 1u);
    li += (sd >> 1) * lm;
    lm *= lat_t;
    stop = stop || (w[d] >> 31);
    mult *= base;
  }
  if (key - hot_lo < hot_n) {
    atomicAdd(hot + (key - hot_lo), 1u);
    return key | STG_HOT;
  }
  if (STAGE && lat) return STG_LAT | li;
  if (!STAGE) atomicAdd(hist + key, 1u);
  return key;
}

// Stage 2 of the staged count: the cold grams of the staged words go to L2
// as REDs, in a pass of their own (interleaved with the columnar stream the
// same REDs run at well under half their standalone rate).  The pass is
// RED-issue bound (lg_throttle), so the two densest blocks are counted in
// shared memory (one CTA per SM) and flushed once: the success lattice
// (STG_LAT words) and, for k = 3, the third-event grams (BEGIN, s_2, s_1,
// s_0), a dense base^3 block.  Both use 16-bit counters packed two per word;
// a counter spills 2^15 to the histogram when it reaches 2^15, so bit 15 of
// a half is a guard that never carries into its neighbour (fewer than 2^15
// increments can land between a half reaching 2^15 and its spill).
constexpr int SH_T = 1024;
constexpr int SH_DENSE_MAX = 40000;  // 16-bit dense-block counters (80 KB)
constexpr int SH_SMEM_MAX = (SH_DENSE_MAX + (int)LAT_MAX) * 2;

// histogram key of success-lattice cell `li` (digits base lat_t, oldest last)
__device__ __forceinline__ uint32_t lat_key(uint32_t li, uint32_t lat_t, uint32_t base, int k) {
  uint32_t key = 0, mult = 1;
  for (int d = 0; d <= k; ++d) {
    key += (2u * (li % lat_t) + 1u) * mult;
    li /= lat_t;
    mult *= base;
  }
  return key;
}

// counter `ci` reached 2^15 (this thread's increment set the guard bit):
// move 2^15 to the histogram (staged word `w` names the gram)
__device__ __noinline__ void spill16(uint32_t* cells, uint32_t ci, uint32_t* hist, uint32_t w,
                                     uint32_t lat_t, uint32_t base, int k) {
  atomicSub(cells + (ci >> 1), 0x8000u << ((ci & 1u) << 4));
  const uint32_t key = (w & STG_LAT) ? lat_key(w & ~STG_LAT, lat_t, base, k) : w;
  atomicAdd(hist + key, 0x8000u);
}

__global__ void __launch_bounds__(SH_T, 1) stage_hist_kernel(const uint32_t* __restrict__ words,
                                                             int64_t n, uint32_t* __restrict__ reps,
                                                             int64_t n_bins, int n_reps,
                                                             uint32_t dlo, uint32_t dn,
                                                             uint32_t lat_t, uint32_t lat_n,
                                                             uint32_t base, int k) {
  extern __shared__ uint32_t cells[];
  const uint32_t n_cells = ((dn + 1) >> 1) + ((lat_n + 1) >> 1);
  for (uint32_t i = threadIdx.x; i < n_cells; i += SH_T) cells[i] = 0;
  __syncthreads();
  // replica per CTA group: a hot bin's updates spread over n_reps addresses
  uint32_t* __restrict__ hist = reps + (int64_t)(blockIdx.x % n_reps) * n_bins;
  const int64_t stride = (int64_t)gridDim.x * SH_T;
  const int64_t t0 = (int64_t)blockIdx.x * SH_T + threadIdx.x;
  const int64_t n4 = n >> 2;
  // one counter space: dense block [0, dn), lattice from loff2 (word aligned)
  const uint32_t loff2 = 2u * ((dn + 1) >> 1);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(cells);
  const uint32_t lat_adj = loff2 - STG_LAT;  // lattice word -> counter index
  auto one = [&](uint32_t w) {
    if (w & STG_HOT) return;
    const bool lw = (w & STG_LAT) != 0;
    const uint32_t ci = w + (lw ? lat_adj : 0u - dlo);
    if (lw || ci < dn) {
      const uint32_t sh = (ci & 1u) << 4;
      uint32_t old;
      asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                   : "=r"(old)
                   : "r"(sbase + ((ci >> 1) << 2)), "r"(1u << sh)
                   : "memory");
      if (((old >> sh) & 0xffffu) == 0x7fffu) spill16(cells, ci, hist, w, lat_t, base, k);
    } else {
      atomicAdd(hist + w, 1u);
    }
  };
  // software-pipelined: the next vector is in flight while this one counts
  const uint4* wv = reinterpret_cast<const uint4*>(words);
  uint4 v = t0 < n4 ? __ldcs(wv + t0) : make_uint4(STG_HOT, STG_HOT, STG_HOT, STG_HOT);
  for (int64_t i = t0; i < n4; i += stride) {
    const uint4 nx = i + stride < n4 ? __ldcs(wv + i + stride)
                                     : make_uint4(STG_HOT, STG_HOT, STG_HOT, STG_HOT);
    one(v.x);
    one(v.y);
    one(v.z);
    one(v.w);
    v = nx;
  }
  for (int64_t i = 4 * n4 + t0; i < n; i += stride) one(words[i]);
  // flush: the CTA pair of a cluster sums its two tables over DSMEM, each
  // CTA flushing half of the counters (half the REDs of a per-CTA flush)
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  const uint32_t cr = cl.block_rank(), cn = cl.num_blocks();
  const uint32_t* peer = cn == 2 ? cl.map_shared_rank(cells, cr ^ 1u) : nullptr;
  auto counter = [&](uint32_t word, uint32_t half) {
    uint32_t v = cells[word];
    if (peer) v += peer[word] & (0xffffu << (half << 4));  // halves stay below 2^16
    return (v >> (half << 4)) & 0xffffu;
  };
  // (a half of one CTA is < 2^15 after the main loop, so the sum of the
  // pair's halves is < 2^16 and never carries out of its half)
  for (uint32_t i = cr * ((dn + 1) >> 1) / cn * 2 + threadIdx.x,
                e = cr + 1 == cn ? dn : (cr + 1) * ((dn + 1) >> 1) / cn * 2;
       i < e; i += SH_T) {
    const uint32_t c = counter(i >> 1, i & 1u);
    if (c) atomicAdd(hist + dlo + i, c);
  }
  const uint32_t loff = (dn + 1) >> 1;
  for (uint32_t i = cr * ((lat_n + 1) >> 1) / cn * 2 + threadIdx.x,
                e = cr + 1 == cn ? lat_n : (cr + 1) * ((lat_n + 1) >> 1) / cn * 2;
       i < e; i += SH_T) {
    const uint32_t c = counter(loff + (i >> 1), i & 1u);
    if (c) atomicAdd(hist + lat_key(i, lat_t, base, k), c);
  }
  cl.sync();  // the peer's table stays live until both halves are flushed
}

// hist += sum of the replicas (one pass over n_reps * n_bins words in L2)
__global__ void fold_replicas_kernel(const uint32_t* __restrict__ reps, int64_t n_bins, int n_reps,
                                     uint32_t* __restrict__ hist) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_bins;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t acc = 0;
    for (int r = 0; r < n_reps; ++r) acc += __ldcs(reps + (int64_t)r * n_bins + i);
    if (acc) hist[i] += acc;
  }
}

// OUT: 0 = cold grams straight to L2, 1 = same + flagged token stream,
// 2 = staged words to `stage_out` (counted by stage_hist_kernel)
template <int K, int OUT>
__global__ void __launch_bounds__(CT) columnar_count_kernel(const paste_columnar_desc C,
                                                            MineGeom g, uint32_t* __restrict__ hist,
                                                            int32_t* __restrict__ tok_out,
                                                            uint32_t* __restrict__ stage_out,
                                                            unsigned long long* tile_ctr,
                                                            uint32_t hot_lo, uint32_t hot_n,
                                                            uint32_t lat_t) {
  extern __shared__ __align__(16) uint8_t c_smem[];
  ColumnTile* tiles = reinterpret_cast<ColumnTile*>(c_smem);
  uint32_t* hot = reinterpret_cast<uint32_t*>(tiles + CNST);
  __shared__ uint64_t full[CNST], empty[CNST];
  __shared__ int64_t stage_tile[CNST];
  for (uint32_t i = threadIdx.x; i < hot_n; i += CT) hot[i] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CNST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t n = C.n_events;
  const int64_t n_tiles = (n + CTILE - 1) / CTILE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long segs = 0, bad = 0;
  if (warp == CW) {
    // ---- producer: claim tiles until the trace is exhausted -----------------
    for (int it = 0;; ++it) {
      const int st = it % CNST;
      if (it >= CNST) mbar_wait(&empty[st], ((it / CNST) - 1) & 1);
      int64_t t = 0;
      if (lane == 0) t = (int64_t)atomicAdd(tile_ctr, 1ull);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= n_tiles) {
        if (lane == 0) {
          stage_tile[st] = -1;
          mbar_arrive(&full[st]);  // release: consumers see the sentinel
        }
        break;
      }
      if (lane == 0) stage_tile[st] = t;
      produce_tile(C, t, &tiles[st], &full[st], lane);
    }
  } else {
    // ---- consumers -----------------------------------------------------------
    const uint32_t S = (uint32_t)g.S, base = (uint32_t)g.base;
    const double gap = C.inactivity_ms;
    for (int it = 0;; ++it) {
      const int st = it % CNST;
      mbar_wait(&full[st], (it / CNST) & 1);
      const int64_t t = stage_tile[st];
      if (t < 0) break;
      const ColumnTile* T = &tiles[st];
      const int64_t g0 = t * CTILE - CPRE;
      const int l0 = CPRE + warp * 64;  // the warp's first slot
      const int64_t x0 = g0 + l0;
      // lane L owns span events e0 = 2L, e1 = 2L + 1 (slots l, l + 1): one
      // vector load per column for both, scalar loads of the slot before
      const int l = l0 + 2 * lane;
      const int64_t xa = x0 + 2 * lane, xb = xa + 1;
      const int2 sg = *reinterpret_cast<const int2*>(T->sig + l);
      const int2 ss = *reinterpret_cast<const int2*>(T->sess + l);
      const int2 sq = *reinterpret_cast<const int2*>(T->seq + l);
      const double2 ts = *reinterpret_cast<const double2*>(T->ts + l);
      const double2 te = *reinterpret_cast<const double2*>(T->te + l);
      const int32_t ps = T->sess[l - 1], pq = T->seq[l - 1];
      const double pts = T->ts[l - 1], pte = T->te[l - 1];
      uint32_t v0, v1;
      {
        const bool b0 = (ps != ss.x) || (__dsub_rn(ts.x, pte) > gap);
        const bool b1 = (ss.x != ss.y) || (__dsub_rn(ts.y, te.x) > gap);
        v0 = (uint32_t)sg.x | (b0 ? SEG_START : 0u);
        v1 = (uint32_t)sg.y | (b1 ? SEG_START : 0u);
        if (xa <= 0 || xa >= n) v0 = (xa == 0 ? (uint32_t)sg.x : 0u) | SEG_START;
        if (xb >= n) v1 = SEG_START;
      }
      // halo: lanes < K hold the word of slot l0-1-lane (the rest: unused)
      const int hl = lane < K ? -1 - lane : -1;
      const uint32_t h = slot_word(T, l0 + hl, x0 + hl, n, gap);
      constexpr int HU = (K + 1) / 2;
      uint32_t up0[HU + 1], up1[HU + 1], hs[K + 1];
#pragma unroll
      for (int j = 1; j <= HU; ++j) {
        up0[j] = __shfl_up_sync(0xffffffffu, v0, j);
        up1[j] = __shfl_up_sync(0xffffffffu, v1, j);
      }
#pragma unroll
      for (int d = 1; d <= K; ++d) hs[d] = __shfl_sync(0xffffffffu, h, (d - 2 * lane - 1) & 31);
      uint32_t w0[K + 1], w1[K + 1];
      w0[0] = v0;
      w1[0] = v1;
#pragma unroll
      for (int d = 1; d <= K; ++d) {
        // e0 = 2L at distance d: lane L - ceil(d/2), word (d even ? v0 : v1)
        const int c = (d + 1) / 2;
        w0[d] = lane >= c ? ((d & 1) ? up1[c] : up0[d / 2]) : hs[d];
        // e1 = 2L + 1 at distance d: lane L - floor(d/2), word (d odd ? v0 : v1)
        const int f = d / 2;
        w1[d] = d == 1 ? v0 : (lane >= f ? ((d & 1) ? up0[f] : up1[f]) : hs[d - 1]);
      }
      constexpr bool STAGE = OUT == 2;
      uint32_t k0 = 0, k1 = 0;
      if (xa < n) {
        k0 = count_event<K, STAGE>(w0, S, base, hot_lo, hot_n, hot, hist, lat_t);
        segs += v0 >> 31;  // segment starts
        if (xa > 0) {
          const bool back = (ts.x < pts) | ((ts.x == pts) & (sq.x <= pq));
          bad += (ss.x < ps) | ((ss.x == ps) & back);
        }
        if (OUT == 1) tok_out[xa] = (int32_t)v0;
      }
      if (xb < n) {
        k1 = count_event<K, STAGE>(w1, S, base, hot_lo, hot_n, hot, hist, lat_t);
        segs += v1 >> 31;
        const bool back = (ts.y < ts.x) | ((ts.y == ts.x) & (sq.y <= sq.x));
        bad += (ss.y < ss.x) | ((ss.y == ss.x) & back);
        if (OUT == 1) tok_out[xb] = (int32_t)v1;
      }
      if (STAGE) {
        if (xb < n) __stcs(reinterpret_cast<uint2*>(stage_out + xa), make_uint2(k0, k1));
        else if (xa < n) stage_out[xa] = k0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  // flush the hot-gram table
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < hot_n; i += CT)
    if (hot[i]) atomicAdd(hist + hot_lo + i, hot[i]);
  // warp-reduce the counters
  for (int o = 16; o > 0; o >>= 1) {
    segs += __shfl_xor_sync(0xffffffffu, segs, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if (lane == 0) {
    if (C.n_segments && segs) atomicAdd(reinterpret_cast<unsigned long long*>(C.n_segments), segs);
    if (C.n_unsorted && bad) atomicAdd(reinterpret_cast<unsigned long long*>(C.n_unsorted), bad);
  }
}

// One tile counter per stream (reset on the stream before every launch), so
// concurrent launches on different streams never share one.
static unsigned long long* tile_counter(cudaStream_t stream) {
  static std::mutex mu;
  static std::unordered_map<cudaStream_t, unsigned long long*> ctrs;
  std::lock_guard<std::mutex> lock(mu);
  auto it = ctrs.find(stream);
  if (it != ctrs.end()) return it->second;
  unsigned long long* p = nullptr;
  if (cudaMalloc(&p, sizeof(unsigned long long)) != cudaSuccess) return nullptr;
  ctrs[stream] = p;
  return p;
}

template <int K, int OUT>
static int launch_columnar(const paste_columnar_desc& c, const MineGeom& g, uint32_t* hist,
                           uint32_t* stage, int64_t tiles, cudaStream_t stream) {
  // hot grams: positions 2..K all BEGIN (a segment's first two events),
  // dense index s_0 + base * s_1
  uint32_t hot_lo = 0, hot_n = (uint32_t)g.base * (uint32_t)g.base;
  uint32_t pw = hot_n;
  for (int d = 2; d <= K; ++d, pw *= (uint32_t)g.base) hot_lo += (uint32_t)g.S * pw;
  if (hot_n > (uint32_t)CHOT_MAX) hot_n = 0;
  const size_t smem = sizeof(ColumnTile) * CNST + (size_t)CHOT_MAX * sizeof(uint32_t);
  // the attribute is per device context: set it on every call (cheap), so a
  // second GPU in the same process launches too
  cudaFuncSetAttribute(columnar_count_kernel<K, OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  static int grid_cap = 0, sms = 0;
  if (grid_cap == 0) {
    int dev = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, columnar_count_kernel<K, OUT>, CT, smem);
    grid_cap = sms * (occ > 0 ? occ : 1);
  }
  unsigned long long* ctr = tile_counter(stream);
  if (ctr == nullptr) return -2;
  if (cudaMemsetAsync(ctr, 0, sizeof(*ctr), stream) != cudaSuccess) return -2;
  const int64_t grid = tiles < grid_cap ? tiles : grid_cap;
  // success lattice (staged counting): (S/2)^(K+1) cells, keys below 2^30
  uint32_t lat_t = 0, lat_n = 0;
  if (OUT == 2 && g.n_bins <= (int64_t)STG_LAT) {
    uint64_t cells = 1;
    for (int d = 0; d <= K; ++d) cells *= (uint64_t)(g.S / 2);
    if (g.S >= 2 && cells <= LAT_MAX) {
      lat_t = (uint32_t)(g.S / 2);
      lat_n = (uint32_t)cells;
    }
  }
  columnar_count_kernel<K, OUT><<<(unsigned)grid, CT, smem, stream>>>(c, g, hist, c.tokens_out,
                                                                      stage, ctr, hot_lo, hot_n,
                                                                      lat_t);
  count_launch();
  if (OUT == 2) {
    // with the lattice in shared memory the cold REDs are spread enough to go
    // straight into the histogram; otherwise into STG_REPS replicas + fold
    const int n_reps = (lat_n > 0 && getenv("PASTE_STAGE_REPS") == nullptr) ? 1 : STG_REPS;
    uint32_t* reps = n_reps == 1 ? hist : stage + stage_words(c.n_events);
    if (n_reps > 1 &&
        cudaMemsetAsync(reps, 0, (size_t)n_reps * g.n_bins * sizeof(uint32_t), stream) !=
            cudaSuccess)
      return -2;
    // dense block (k = 3): grams whose oldest symbol is BEGIN -- a segment's
    // third event -- when their base^3 counters fit in shared memory
    uint32_t dlo = 0, dn = 0;
    const uint64_t b3 = (uint64_t)g.base * g.base * g.base;
    if (K == 3 && b3 <= (uint64_t)SH_DENSE_MAX) {
      dlo = (uint32_t)((uint64_t)g.S * b3);
      dn = (uint32_t)b3;
    }
    cudaFuncSetAttribute(stage_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SH_SMEM_MAX);  // per device context: every call
    const size_t sh_bytes = (size_t)(((dn + 1) >> 1) + ((lat_n + 1) >> 1)) * sizeof(uint32_t);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr_c[1];
    attr_c[0].id = cudaLaunchAttributeClusterDimension;
    attr_c[0].val.clusterDim.x = 2;  // CTA pairs (148 SMs = 74 pairs)
    attr_c[0].val.clusterDim.y = 1;
    attr_c[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(sms & ~1));
    cfg.blockDim = dim3(SH_T);
    cfg.dynamicSmemBytes = sh_bytes;
    cfg.stream = stream;
    cfg.attrs = attr_c;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, stage_hist_kernel, (const uint32_t*)stage, (int64_t)c.n_events,
                           reps, (int64_t)g.n_bins, n_reps, dlo, dn, lat_t, lat_n,
                           (uint32_t)g.base, (int)K) != cudaSuccess)
      return -2;
    count_launch();
    if (n_reps > 1) {
      fold_replicas_kernel<<<(unsigned)(sms * 4), 256, 0, stream>>>(reps, g.n_bins, n_reps, hist);
      count_launch();
    }
  }
  return 0;
}

static int ingest_count_impl(const paste_columnar_desc* c, const paste_mine_desc* d,
                             uint32_t* stage, void* stream) {
  reset_launches();
  PASTE_REQUIRE(c != nullptr && d != nullptr, "null descriptor");
  MineGeom g;
  if (make_geom(d->n_sigs, d->k, &g) != 0 || d->k + 1 > CPRE) {
    set_error("mining geometry out of range (n_sigs=%d, k=%d)", d->n_sigs, d->k);
    return PASTE_ERR_UNSUPPORTED;
  }
  if (c->n_events == 0) return PASTE_OK;
  const uintptr_t mis = (uintptr_t)c->session | (uintptr_t)c->seq | (uintptr_t)c->t_start |
                        (uintptr_t)c->t_end | (uintptr_t)c->sig;
  PASTE_REQUIRE((mis & 15) == 0, "columnar arrays must be 16-byte aligned");
  PASTE_REQUIRE(stage == nullptr || ((uintptr_t)stage & 15) == 0,
                "staging buffer must be 16-byte aligned");
  const int64_t tiles = (c->n_events + CTILE - 1) / CTILE;
  // staged counting needs gram keys below 2^30 (two flag bits)
  const int out = c->tokens_out != nullptr ? 1
                  : (stage != nullptr && g.n_bins <= (int64_t)STG_KEY + 1) ? 2 : 0;
  int rc = -1;
#define PASTE_COLUMNAR(KV)                                                                        \
  if (d->k == KV) {                                                                               \
    if (out == 1) rc = launch_columnar<KV, 1>(*c, g, d->hist, stage, tiles, (cudaStream_t)stream); \
    else if (out == 2)                                                                            \
      rc = launch_columnar<KV, 2>(*c, g, d->hist, stage, tiles, (cudaStream_t)stream);            \
    else rc = launch_columnar<KV, 0>(*c, g, d->hist, stage, tiles, (cudaStream_t)stream);         \
  }
  PASTE_COLUMNAR(1) PASTE_COLUMNAR(2) PASTE_COLUMNAR(3) PASTE_COLUMNAR(4) PASTE_COLUMNAR(5)
  PASTE_COLUMNAR(6)
#undef PASTE_COLUMNAR
  if (rc == -2) {
    set_error("could not allocate the columnar tile counter");
    return PASTE_ERR_CUDA;
  }
  if (rc != 0) {
    set_error("k=%d outside the columnar kernel's range", d->k);
    return PASTE_ERR_UNSUPPORTED;
  }
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

extern "C" int paste_mine_ingest_count(const paste_columnar_desc* c, const paste_mine_desc* d,
                                       void* stream) {
  return ingest_count_impl(c, d, nullptr, stream);
}

extern "C" int64_t paste_mine_stage_bytes(int64_t n_events, int32_t n_sigs, int32_t k) {
  MineGeom g;
  if (n_events <= 0 || make_geom(n_sigs, k, &g) != 0) return 0;
  return (stage_words(n_events) + (int64_t)STG_REPS * g.n_bins) * 4;
}

extern "C" int paste_mine_ingest_count_staged(const paste_columnar_desc* c,
                                              const paste_mine_desc* d, void* stage,
                                              int64_t stage_bytes, void* stream) {
  PASTE_REQUIRE(c != nullptr && d != nullptr, "null descriptor");
  PASTE_REQUIRE(stage == nullptr || stage_bytes >= paste_mine_stage_bytes(c->n_events, d->n_sigs, d->k),
                "staging buffer too small");
  return ingest_count_impl(c, d, reinterpret_cast<uint32_t*>(stage), stream);
}

extern "C" int64_t paste_mine_sort_scratch_bytes(int64_t cap) {
  return cap <= 0 ? 0 : cap * (int64_t)(sizeof(SelRow) + sizeof(ulonglong2) + sizeof(uint32_t));
}

extern "C" int paste_mine_select_sorted(const paste_mine_desc* d, int64_t sigma, double tau,
                                        int64_t cap, uint64_t* n_out, int64_t* out, void* scratch,
                                        void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr && n_out != nullptr && out != nullptr && scratch != nullptr,
                "null argument");
  PASTE_REQUIRE(cap > 0 && cap < ((int64_t)1 << 31), "capacity out of range");
  MineGeom g;
  if (make_geom(d->n_sigs, d->k, &g) != 0) {
    set_error("mining geometry out of range (n_sigs=%d, k=%d)", d->n_sigs, d->k);
    return PASTE_ERR_UNSUPPORTED;
  }
  cudaStream_t st = (cudaStream_t)stream;
  SelRow* rows = reinterpret_cast<SelRow*>(scratch);
  ulonglong2* keys = reinterpret_cast<ulonglong2*>(rows + cap);
  uint32_t* rank = reinterpret_cast<uint32_t*>(keys + cap);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(n_out);
  PASTE_CUDA_CHECK(cudaMemsetAsync(n_out, 0, sizeof(uint64_t), st));
  PASTE_CUDA_CHECK(cudaMemsetAsync(rank, 0, (size_t)cap * sizeof(uint32_t), st));
  const int64_t total = (int64_t)g.T * g.n_ctx;
  select_keyed_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      g, U64(d->tool_count), U64(d->support), U64(d->match), U64(d->follow), sigma, tau, cap, cnt,
      rows, keys);
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  rank_keys_kernel<<<(unsigned)(sms * 8), RI, 0, st>>>(keys, cnt, cap, rank);
  scatter_rows_kernel<<<(unsigned)(sms * 2), 256, 0, st>>>(rows, rank, cnt, cap,
                                                          reinterpret_cast<SelRow*>(out));
  count_launch(3);
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
