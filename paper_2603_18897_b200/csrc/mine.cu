// K2 count_structural / K1 ingest / mining selection for sm_100a.
//
// Reference: mine() (mining.py:248-292) with its windows and distinct-
// subsequence support (mining.py:164-194, 266-275), anchored / contiguous
// matching (match_at, mining.py:119-156) and the per-context rescans of
// _collect_occurrences (mining.py:215-227).
//
// Reformulation (verified exact): every count mine()
// needs is a function of one (k+1)-gram of a session's tool tokens.  For
// position j of a stream s_0..s_{L-1} (j = L is the END position),
// T_j = (s_{j-k} .. s_{j-1}, s_j) with BEGIN before the stream and END after
// it:
//   * target j (j < L): window = the non-BEGIN part of (s_{j-k}..s_{j-1});
//     support[tool(s_j)][c] += 1 for each distinct subsequence c (anchored)
//     or suffix c (contiguous);
//   * anchor a = j-1 (s_{j-1} != BEGIN): the contexts that match at a are
//     u + (s_a) for each distinct subsequence u of the non-BEGIN part of
//     (s_{j-k}..s_{j-2}) (anchored, rightmost embedding is complete) or the
//     contiguous suffixes ending at a; match[c] += 1 and, when j < L,
//     follow[c][tool(s_j)] += 1.
// So the device counts one histogram H over (k+1)-grams (one warp-aggregated
// increment per position) and expands the non-zero bins once.
//
// Token stream format: int32 sig ids with bit 31 set on the first token of
// every segment (session after gap splitting).
#include "common.cuh"

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
// count: one (k+1)-gram per token plus one END gram per segment
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
  // END gram after the last token of a segment
  const bool last = (i + 1 == n) || (__ldg(tok + i + 1) & SEG_START);
  if (last) {
    int64_t kend = g.S + 1;  // END at d = 0
    int64_t mul = g.base;
    bool st = false;
    for (int d = 1; d <= g.k; ++d) {
      int sym = g.S;
      if (!st) {
        const uint32_t p = __ldg(tok + i - (d - 1));
        sym = (int)(p & ~SEG_START);
        st = (p & SEG_START) != 0;
      }
      kend += (int64_t)sym * mul;
      mul *= g.base;
    }
    atomicAdd(hist + kend, 1u);
  }
}

// ---------------------------------------------------------------------------
// expand: non-zero (k+1)-gram bins -> tool_count / support / match / follow
// ---------------------------------------------------------------------------
__device__ __forceinline__ int distinct_subseqs(const int* w, int n, int* out, int* out_len,
                                                int max_out, bool include_empty, int maxlen) {
  // all order-preserving subsequences of w (length n), deduplicated
  int cnt = 0;
  for (int mask = include_empty ? 0 : 1; mask < (1 << n); ++mask) {
    int c[8], len = 0;
    for (int i = 0; i < n; ++i)
      if (mask & (1 << i)) c[len++] = w[i];
    bool dup = false;
    for (int q = 0; q < cnt && !dup; ++q) {
      if (out_len[q] != len) continue;
      bool same = true;
      for (int i = 0; i < len; ++i) same &= out[q * maxlen + i] == c[i];
      dup = same;
    }
    if (dup || cnt >= max_out) continue;
    for (int i = 0; i < len; ++i) out[cnt * maxlen + i] = c[i];
    out_len[cnt++] = len;
  }
  return cnt;
}

__global__ void expand_grams_kernel(const uint32_t* __restrict__ hist, MineGeom g, int relation,
                                    unsigned long long* tool_count, unsigned long long* support,
                                    unsigned long long* match, unsigned long long* follow) {
  const int64_t key = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (key >= g.n_bins) return;
  const uint32_t h = hist[key];
  if (h == 0) return;
  int sym[17];  // sym[d] = s_{j-d}
  {
    int64_t k2 = key;
    for (int d = 0; d <= g.k; ++d) {
      sym[d] = (int)(k2 % g.base);
      k2 /= g.base;
    }
  }
  const int BEGIN = g.S, END = g.S + 1;
  const int s0 = sym[0];
  // window before target j: (s_{j-k}..s_{j-1}) minus BEGINs, oldest first
  int win[16], wl = 0;
  for (int d = g.k; d >= 1; --d)
    if (sym[d] != BEGIN) win[wl++] = sym[d];
  int subs[64 * 6], sub_len[64];  // k <= 6: at most 2^6 subsequences
  if (s0 != END) {  // target occurrence
    const int tool = s0 >> 1;
    atomicAdd(tool_count + tool, (unsigned long long)h);
    if (relation == PASTE_REL_ANCHORED) {
      const int ns = distinct_subseqs(win, wl, subs, sub_len, 64, false, 6);
      for (int q = 0; q < ns; ++q)
        atomicAdd(support + (int64_t)tool * g.n_ctx + ctx_index(g, subs + q * 6, sub_len[q]),
                  (unsigned long long)h);
    } else {
      for (int st = 0; st < wl; ++st)
        atomicAdd(support + (int64_t)tool * g.n_ctx + ctx_index(g, win + st, wl - st),
                  (unsigned long long)h);
    }
  }
  if (sym[1] == BEGIN || sym[1] == END) return;  // no anchor at j-1
  // anchor a = j-1; previous k-1 events (s_{j-k}..s_{j-2}) minus BEGINs
  int prev[16], pl = 0;
  for (int d = g.k; d >= 2; --d)
    if (sym[d] != BEGIN) prev[pl++] = sym[d];
  const int follow_tool = s0 != END ? (s0 >> 1) : -1;
  if (relation == PASTE_REL_ANCHORED) {
    const int ns = distinct_subseqs(prev, pl, subs, sub_len, 64, true, 6);
    for (int q = 0; q < ns; ++q) {
      int c[16];
      const int len = sub_len[q];
      for (int i = 0; i < len; ++i) c[i] = subs[q * 6 + i];
      c[len] = sym[1];
      const int64_t ci = ctx_index(g, c, len + 1);
      atomicAdd(match + ci, (unsigned long long)h);
      if (follow_tool >= 0) atomicAdd(follow + ci * g.T + follow_tool, (unsigned long long)h);
    }
  } else {
    int c[16];
    for (int len = 1; len <= pl + 1; ++len) {  // suffixes ending at the anchor
      for (int i = 0; i < len - 1; ++i) c[i] = prev[pl - (len - 1) + i];
      c[len - 1] = sym[1];
      const int64_t ci = ctx_index(g, c, len);
      atomicAdd(match + ci, (unsigned long long)h);
      if (follow_tool >= 0) atomicAdd(follow + ci * g.T + follow_tool, (unsigned long long)h);
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
  const int threads = 128;
  expand_grams_kernel<<<(unsigned)((g.n_bins + threads - 1) / threads), threads, 0,
                        (cudaStream_t)stream>>>(d->hist, g, d->relation, U64(d->tool_count),
                                                U64(d->support), U64(d->match), U64(d->follow));
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
