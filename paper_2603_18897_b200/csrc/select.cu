// K6 admission_select: greedy_speculative_selection on the device.
//
// Reference (scheduling.py:59-60, 242-258): U = (p * T) / (c * d) in fp64;
// jobs are visited in ascending (-U, -p, id) and taken while their cost fits
// both the remaining slack and the remaining budget; both decrease by the
// job's cost, so the test is cost <= cap with cap = min(slack, budget)
// decreasing by each selected cost.
//
// Device plan (cost >= 1):
//   * once a job of cost c is rejected, cap < c for good, so the selected
//     jobs of cost c are a PREFIX (in key order) of at most floor(cap0 / c)
//     jobs of that cost -- the only candidates;
//   * a radix select over the full 192-bit key (-U, -p, id), 8 bits per pass
//     with a per-class early exit, finds for every cost class c <= cap0 the
//     key of its floor(cap0/c)-th best job; the jobs at or below their class
//     threshold are exactly the candidates (ids are unique, so no ties);
//   * the candidates are sorted by the full key (-U, -p, id) in shared memory
//     (bitonic) and one warp runs the greedy scan; visiting a superset of the
//     selected jobs in the same relative order yields the same decisions.
#include <cub/cub.cuh>

#include "common.cuh"

namespace paste {

constexpr int SEL_MAX_CAP = 64;       // cost classes handled by the radix select
constexpr int SEL_MAX_CAND = 4096;    // candidates sorted in one CTA
constexpr int SEL_T = 256;

__device__ __forceinline__ uint64_t desc_key(double v) {
  // ascending order of the returned key == descending order of v (v != NaN);
  // -0.0 and 0.0 compare equal in the reference, so they share a key
  if (v == 0.0) v = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~asc;
}

struct SelJob {
  uint64_t ku;  // -U order key
  uint64_t kp;  // -p order key
  int64_t id;
  int32_t cost;
  int32_t idx;
};

__device__ __forceinline__ bool sel_less(const SelJob& a, const SelJob& b) {
  if (a.ku != b.ku) return a.ku < b.ku;
  if (a.kp != b.kp) return a.kp < b.kp;
  if (a.id != b.id) return a.id < b.id;
  return a.idx < b.idx;  // sorted() is stable: equal keys keep the input order
}

// per-job keys + validation
__global__ void sel_keys_kernel(paste_select_desc D, uint64_t* ku, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n_jobs) return;
  const double p = D.p[i], c = (double)D.cost[i], d = D.duration[i];
  const double u = __ddiv_rn(__dmul_rn(p, D.benefit[i]), __dmul_rn(c, d));
  if (D.cost[i] < 1 || d == 0.0 || u != u || p != p) atomicOr(bad, 1);
  ku[i] = desc_key(u);
}

// The radix select runs over the full 192-bit key (-U, -p, id) so the
// candidate set is exact (ties never inflate it).  Key words: w0 = order key
// of -U, w1 = order key of -p, w2 = id in unsigned order.
__device__ __forceinline__ uint64_t key_word(const paste_select_desc& D, const uint64_t* ku,
                                             int64_t i, int w) {
  if (w == 0) return ku[i];
  if (w == 1) return desc_key(D.p[i]);
  return (uint64_t)D.id[i] ^ 0x8000000000000000ull;
}

// per cost class: histogram of digit `pass` among jobs matching the prefix
__global__ void sel_hist_kernel(paste_select_desc D, const uint64_t* ku, int cap, int pass,
                                const uint64_t* prefix, const int* done, const int* all_done,
                                unsigned* hist) {
  if (*all_done) return;
  extern __shared__ unsigned h[];  // cap x 256 digit counters
  for (int i = threadIdx.x; i < cap * 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int word = pass >> 3, shift = 56 - 8 * (pass & 7);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D.n_jobs;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = D.cost[i];
    if (c < 1 || c > cap || done[c - 1]) continue;
    const uint64_t* pf = prefix + 3 * (c - 1);
    bool match = true;
    for (int w = 0; w < word && match; ++w) match = key_word(D, ku, i, w) == pf[w];
    if (!match) continue;
    const uint64_t k = key_word(D, ku, i, word);
    if (shift < 56 && (k >> (shift + 8)) != (pf[word] >> (shift + 8))) continue;
    atomicAdd(&h[(c - 1) * 256 + (int)((k >> shift) & 255)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cap * 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// locate the rank-th job's digit; a class is done when its bucket holds a
// single job (or the class has fewer jobs than its quota): the threshold
// then covers the rest of that bucket with all-ones low bits
__global__ void sel_pick_kernel(int cap, int pass, uint64_t* prefix, int64_t* rank, unsigned* hist,
                                int* done, int* all_done) {
  const int c = threadIdx.x + 1;
  __shared__ int remaining;
  if (threadIdx.x == 0) remaining = 0;
  __syncthreads();
  if (c <= cap && !*all_done) {
    unsigned* h = hist + (c - 1) * 256;
    uint64_t* pf = prefix + 3 * (c - 1);
    const int word = pass >> 3, shift = 56 - 8 * (pass & 7);
    if (!done[c - 1]) {
      const int64_t r = rank[c - 1];
      int64_t acc = 0;
      int digit = -1;
      for (int dg = 0; dg < 256; ++dg) {
        if (acc + h[dg] > r) { digit = dg; break; }
        acc += h[dg];
      }
      if (digit < 0) {  // fewer jobs than floor(cap/c): the whole class
        done[c - 1] = 1;
        pf[0] = pf[1] = pf[2] = ~0ull;
      } else {
        rank[c - 1] = r - acc;
        const uint64_t low = shift == 0 ? 0ull : ((1ull << shift) - 1);
        pf[word] = (pf[word] & ~(0xffull << shift)) | ((uint64_t)digit << shift);
        if (h[digit] == 1 || pass == 23) {  // unique: close the threshold
          done[c - 1] = 1;
          pf[word] |= low;
          for (int w = word + 1; w < 3; ++w) pf[w] = ~0ull;
        }
      }
    }
    for (int dg = 0; dg < 256; ++dg) h[dg] = 0;
    if (!done[c - 1]) atomicAdd(&remaining, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0 && remaining == 0) *all_done = 1;
}

// candidates: class jobs whose full key is <= the class threshold
__global__ void sel_compact_kernel(paste_select_desc D, const uint64_t* ku, int cap,
                                   const uint64_t* thresh, unsigned* n_cand, int32_t* cand) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n_jobs) return;
  const int c = D.cost[i];
  if (c < 1 || c > cap) return;
  const uint64_t* t = thresh + 3 * (c - 1);
  bool le = true;
  for (int w = 0; w < 3; ++w) {
    const uint64_t k = key_word(D, ku, i, w);
    if (k != t[w]) {
      le = k < t[w];
      break;
    }
  }
  if (!le) return;
  const unsigned s = atomicAdd(n_cand, 1u);
  if (s < (unsigned)SEL_MAX_CAND) cand[s] = (int32_t)i;
}

// one CTA: sort the candidates by (-U, -p, id) and run the greedy scan
__global__ void __launch_bounds__(1024) sel_greedy_kernel(paste_select_desc D, const uint64_t* ku,
                                                          const unsigned* n_cand_p,
                                                          const int32_t* cand, int64_t slack,
                                                          int64_t budget, int* status) {
  extern __shared__ SelJob sj[];
  const unsigned n_cand = *n_cand_p;
  if (n_cand > (unsigned)SEL_MAX_CAND) {
    if (threadIdx.x == 0) *status = 1;  // outside the envelope
    return;
  }
  int P = 1;
  while (P < (int)n_cand) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    SelJob j;
    if (i < (int)n_cand) {
      const int32_t x = cand[i];
      j.ku = ku[x];
      j.kp = desc_key(D.p[x]);
      j.id = D.id[x];
      j.cost = D.cost[x];
      j.idx = x;
    } else {
      j.ku = ~0ull;
      j.kp = ~0ull;
      j.id = INT64_MAX;
      j.cost = 0;
      j.idx = -1;
    }
    sj[i] = j;
  }
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)  // bitonic sort
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ jj;
        if (l > i) {
          const bool up = (i & k) == 0;
          const SelJob a = sj[i], b = sj[l];
          if (sel_less(b, a) == up) {
            sj[i] = b;
            sj[l] = a;
          }
        }
      }
      __syncthreads();
    }
  if (threadIdx.x == 0) {
    int64_t r = slack, b = budget;
    int64_t n_sel = 0;
    for (int i = 0; i < (int)n_cand; ++i) {
      const int64_t c = sj[i].cost;
      if (c <= r && c <= b) {
        D.selected[n_sel++] = sj[i].idx;
        r -= c;
        b -= c;
      }
    }
    *D.n_selected = n_sel;
    *status = 0;
  }
}


// ---------------------------------------------------------------------------
// General path (any min(slack, budget), any number of ties): a full device
// sort by (-U, -p, id) of the jobs that can ever fit (cost <= cap), a stable
// sort of those by cost to rank each job inside its cost class, the same
// floor(cap / c) prefix rule per class to keep the candidates, and a
// warp-parallel greedy scan over the candidates in key order.
// ---------------------------------------------------------------------------
__global__ void gen_keys_kernel(paste_select_desc D, const uint64_t* ku, int64_t cap,
                                uint64_t* k0, uint64_t* k1, uint64_t* k2, uint8_t* fit,
                                int32_t* iota) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n_jobs) return;
  const int c = D.cost[i];
  fit[i] = c >= 1 && (int64_t)c <= cap;
  k0[i] = ku[i];
  k1[i] = desc_key(D.p[i]);
  k2[i] = (uint64_t)D.id[i] ^ 0x8000000000000000ull;
  iota[i] = (int32_t)i;
}

__global__ void gen_cost_kernel(paste_select_desc D, const int32_t* order, int64_t n,
                                int32_t* ckey, int32_t* pos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  ckey[i] = D.cost[order[i]];
  pos[i] = (int32_t)i;
}

// t-th element of the cost-sorted array: rank inside its class = t - first
// index of its cost (binary search); candidate if rank < floor(cap / c)
__global__ void gen_flag_kernel(const int32_t* csorted, const int32_t* pos_sorted, int64_t n,
                                int64_t cap, uint8_t* flag) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int32_t c = csorted[t];
  int64_t lo = 0, hi = t;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (csorted[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  flag[pos_sorted[t]] = (t - lo) < cap / c ? 1 : 0;
}

__global__ void gen_gather_kernel(const uint64_t* src, const int32_t* order, int64_t n,
                                  uint64_t* dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[order[i]];
}

__global__ void gen_iota_kernel(int32_t* a, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int32_t)i;
}

// one warp: greedy over the candidates (positions in key order, ascending)
__global__ void gen_scan_kernel(paste_select_desc D, const int32_t* order, const int32_t* cand,
                                const int* n_cand_p, int64_t slack, int64_t budget) {
  const int lane = threadIdx.x;
  const int64_t n_cand = *n_cand_p;
  int64_t r = slack, b = budget, n_sel = 0;
  for (int64_t base = 0; base < n_cand; base += 32) {
    if (r < 1 || b < 1) break;  // every cost is >= 1
    const int64_t i = base + lane;
    int32_t job = -1;
    int64_t c = INT64_MAX;
    if (i < n_cand) {
      job = order[cand[i]];
      c = D.cost[job];
    }
    bool alive = i < n_cand;
    for (;;) {
      const unsigned m = __ballot_sync(0xffffffffu, alive && c <= r && c <= b);
      if (!m) break;
      const int f = __ffs(m) - 1;
      const int64_t cf = __shfl_sync(0xffffffffu, c, f);
      const int32_t jf = __shfl_sync(0xffffffffu, job, f);
      if (lane == 0) D.selected[n_sel] = jf;
      ++n_sel;
      r -= cf;
      b -= cf;
      alive = alive && lane > f;
    }
  }
  if (lane == 0) *D.n_selected = n_sel;
}
}  // namespace paste

using namespace paste;

static int64_t align256(int64_t b) { return (b + 255) / 256 * 256; }

static size_t general_cub_bytes(int64_t n) {
  const int m = (int)(n > 0 ? n : 1);
  size_t a = 0, b = 0, c = 0;
  cub::DoubleBuffer<uint64_t> k64(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> v32(nullptr, nullptr), k32(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, k64, v32, m);
  cub::DeviceRadixSort::SortPairs(nullptr, b, k32, v32, m);
  cub::DeviceSelect::Flagged(nullptr, c, (int32_t*)nullptr, (uint8_t*)nullptr, (int32_t*)nullptr,
                             (int*)nullptr, m);
  return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

// bytes of the radix-select path (ku first: the general path reuses it)
static int64_t fast_bytes(int64_t n) {
  return align256(8 * n) + 32 * SEL_MAX_CAP + 4 * SEL_MAX_CAP * 256 + 4 * (SEL_MAX_CAP + 4) + 16 +
         4 * SEL_MAX_CAND + 256;
}

static int64_t general_bytes(int64_t n) {
  return 3 * align256(8 * n) + 2 * align256(8 * n) + 2 * align256(4 * n) + align256(n) +
         align256(4 * n) + 256 + (int64_t)general_cub_bytes(n) + 256;
}

// The general path: see gen_* above.  ku = per-job -U order keys (computed).
static int select_general(paste_select_desc* d, int64_t slack, int64_t budget, int64_t cap,
                          const uint64_t* ku, uint8_t* s, uint8_t* s_end, cudaStream_t stream) {
  const int64_t n = d->n_jobs;
  uint64_t* k0 = reinterpret_cast<uint64_t*>(s); s += align256(8 * n);
  uint64_t* k1 = reinterpret_cast<uint64_t*>(s); s += align256(8 * n);
  uint64_t* k2 = reinterpret_cast<uint64_t*>(s); s += align256(8 * n);
  uint64_t* ka = reinterpret_cast<uint64_t*>(s); s += align256(8 * n);
  uint64_t* kb = reinterpret_cast<uint64_t*>(s); s += align256(8 * n);
  int32_t* va = reinterpret_cast<int32_t*>(s); s += align256(4 * n);
  int32_t* vb = reinterpret_cast<int32_t*>(s); s += align256(4 * n);
  uint8_t* flag = s; s += align256(n);
  int32_t* cand = reinterpret_cast<int32_t*>(s); s += align256(4 * n);
  unsigned* counters = reinterpret_cast<unsigned*>(s); s += 256;
  void* tmp = s;
  size_t tmp_bytes = (size_t)(s_end - s);
  PASTE_CUDA_CHECK(cudaMemsetAsync(counters, 0, 16, stream));
  const int blocks = (int)((n + SEL_T - 1) / SEL_T);
  // the jobs that can ever fit, compacted in input order (equal keys must
  // keep it: sorted() is stable)
  gen_keys_kernel<<<blocks, SEL_T, 0, stream>>>(*d, ku, cap, k0, k1, k2, flag, cand);
  count_launch();
  int* n_fit = reinterpret_cast<int*>(counters);
  PASTE_CUDA_CHECK(cub::DeviceSelect::Flagged(tmp, tmp_bytes, cand, flag, va, n_fit, (int)n, stream));
  count_launch(2);
  int h_fit = 0;
  PASTE_CUDA_CHECK(cudaMemcpyAsync(&h_fit, n_fit, 4, cudaMemcpyDeviceToHost, stream));
  PASTE_CUDA_CHECK(cudaStreamSynchronize(stream));
  const int m = h_fit;
  if (m == 0) {
    PASTE_CUDA_CHECK(cudaMemsetAsync(d->n_selected, 0, sizeof(int64_t), stream));
    return PASTE_OK;
  }
  const int mblocks = (m + SEL_T - 1) / SEL_T;
  // LSD over the key words (stable): id, then -p, then -U; values = job index
  cub::DoubleBuffer<int32_t> vals(va, vb);
  const uint64_t* words[3] = {k2, k1, k0};
  for (int w = 0; w < 3; ++w) {
    gen_gather_kernel<<<mblocks, SEL_T, 0, stream>>>(words[w], vals.Current(), m, ka);
    count_launch();
    cub::DoubleBuffer<uint64_t> keys(ka, kb);
    PASTE_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, vals, m, 0, 64, stream));
    count_launch(8);
  }
  // order[t] = job index of the t-th fit job in key order
  const int32_t* order = vals.Current();
  // rank inside each cost class: stable sort of key positions by cost
  int32_t* ck = reinterpret_cast<int32_t*>(ka);
  int32_t* ck2 = reinterpret_cast<int32_t*>(ka) + m;
  int32_t* pos = reinterpret_cast<int32_t*>(kb);
  int32_t* pos2 = reinterpret_cast<int32_t*>(kb) + m;
  gen_cost_kernel<<<mblocks, SEL_T, 0, stream>>>(*d, order, m, ck, pos);
  count_launch();
  int cbits = 1;
  while (cbits < 31 && (int64_t(1) << cbits) <= cap) ++cbits;
  cub::DoubleBuffer<int32_t> ckeys(ck, ck2), cpos(pos, pos2);
  PASTE_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ckeys, cpos, m, 0, cbits, stream));
  count_launch(4);
  gen_flag_kernel<<<mblocks, SEL_T, 0, stream>>>(ckeys.Current(), cpos.Current(), m, cap, flag);
  count_launch();
  // candidate key positions in ascending order
  int32_t* iota = reinterpret_cast<int32_t*>(ckeys.Alternate());
  gen_iota_kernel<<<mblocks, SEL_T, 0, stream>>>(iota, m);
  count_launch();
  int* n_cand = reinterpret_cast<int*>(counters + 1);
  PASTE_CUDA_CHECK(cub::DeviceSelect::Flagged(tmp, tmp_bytes, iota, flag, cand, n_cand, m, stream));
  count_launch(2);
  gen_scan_kernel<<<1, 32, 0, stream>>>(*d, order, cand, n_cand, slack, budget);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  PASTE_CUDA_CHECK(cudaStreamSynchronize(stream));
  return PASTE_OK;
}

extern "C" int paste_select_greedy(paste_select_desc* d, int64_t slack, int64_t budget,
                                   void* scratch, int64_t scratch_bytes, void* stream_) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null descriptor");
  cudaStream_t stream = (cudaStream_t)stream_;
  const int64_t n = d->n_jobs;
  const int64_t cap64 = slack < budget ? slack : budget;
  const int64_t need = paste_select_scratch_bytes(n);
  PASTE_REQUIRE(scratch != nullptr && scratch_bytes >= need, "scratch too small (%lld bytes)",
                (long long)need);
  PASTE_REQUIRE(n < (1ll << 31) - 1, "more than 2^31 - 2 jobs");
  if (n == 0 || cap64 < 1) {
    PASTE_CUDA_CHECK(cudaMemsetAsync(d->n_selected, 0, sizeof(int64_t), stream));
    return PASTE_OK;  // nothing fits (every cost >= 1)
  }
  uint8_t* s0 = static_cast<uint8_t*>(scratch);
  uint8_t* s = s0;
  uint64_t* ku = reinterpret_cast<uint64_t*>(s);
  s += align256(8 * n);
  uint64_t* prefix = reinterpret_cast<uint64_t*>(s);
  s += 24 * SEL_MAX_CAP;
  int64_t* rank = reinterpret_cast<int64_t*>(s);
  s += 8 * SEL_MAX_CAP;
  unsigned* hist = reinterpret_cast<unsigned*>(s);
  s += 4 * SEL_MAX_CAP * 256;
  int* flags = reinterpret_cast<int*>(s);  // [0] bad, [1] status, [2] all done, [3..] done
  s += 4 * (SEL_MAX_CAP + 4);
  unsigned* n_cand = reinterpret_cast<unsigned*>(s);
  s += 16;
  int32_t* cand = reinterpret_cast<int32_t*>(s);
  uint8_t* gen = s0 + fast_bytes(n);
  uint8_t* gen_end = s0 + scratch_bytes;

  PASTE_CUDA_CHECK(cudaMemsetAsync(flags, 0, 4 * (SEL_MAX_CAP + 4), stream));
  const int blocks = (int)((n + SEL_T - 1) / SEL_T);
  sel_keys_kernel<<<blocks, SEL_T, 0, stream>>>(*d, ku, flags);
  count_launch();
  int h_flags[2] = {0, 0};
  if (cap64 > SEL_MAX_CAP) {  // outside the radix-select envelope: general path
    PASTE_CUDA_CHECK(cudaMemcpyAsync(h_flags, flags, sizeof(h_flags), cudaMemcpyDeviceToHost, stream));
    PASTE_CUDA_CHECK(cudaStreamSynchronize(stream));
    if (h_flags[0]) {
      set_error("jobs need cost >= 1, a non-zero duration and a non-NaN utility");
      return PASTE_ERR_INVALID;
    }
    return select_general(d, slack, budget, cap64, ku, gen, gen_end, stream);
  }
  const int cap = (int)cap64;
  // host-side init of the small state (ranks = floor(cap / c) - 1)
  {
    uint64_t h_prefix[3 * SEL_MAX_CAP];
    int64_t h_rank[SEL_MAX_CAP];
    for (int c = 1; c <= SEL_MAX_CAP; ++c) {
      h_prefix[3 * (c - 1)] = h_prefix[3 * (c - 1) + 1] = h_prefix[3 * (c - 1) + 2] = 0;
      h_rank[c - 1] = c <= cap ? cap / c - 1 : 0;
    }
    PASTE_CUDA_CHECK(cudaMemcpyAsync(prefix, h_prefix, sizeof(h_prefix), cudaMemcpyHostToDevice, stream));
    PASTE_CUDA_CHECK(cudaMemcpyAsync(rank, h_rank, sizeof(h_rank), cudaMemcpyHostToDevice, stream));
    PASTE_CUDA_CHECK(cudaMemsetAsync(hist, 0, 4 * SEL_MAX_CAP * 256, stream));
    PASTE_CUDA_CHECK(cudaMemsetAsync(n_cand, 0, 16, stream));
    // a synchronous copy keeps the stack arrays alive until they are consumed
    PASTE_CUDA_CHECK(cudaStreamSynchronize(stream));
  }
  const int hblocks = blocks < 148 * 4 ? blocks : 148 * 4;
  // the shared-memory opt-in is per device: set it on every call (cheap)
  PASTE_CUDA_CHECK(cudaFuncSetAttribute(sel_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        4 * SEL_MAX_CAP * 256));
  PASTE_CUDA_CHECK(cudaFuncSetAttribute(sel_greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)sizeof(SelJob) * SEL_MAX_CAND));
  for (int pass = 0; pass < 24; ++pass) {  // kernels return at once when every class is done
    sel_hist_kernel<<<hblocks, SEL_T, 4 * cap * 256, stream>>>(*d, ku, cap, pass, prefix,
                                                                flags + 3, flags + 2, hist);
    sel_pick_kernel<<<1, SEL_MAX_CAP, 0, stream>>>(cap, pass, prefix, rank, hist, flags + 3,
                                                   flags + 2);
    count_launch(2);
  }
  sel_compact_kernel<<<blocks, SEL_T, 0, stream>>>(*d, ku, cap, prefix, n_cand, cand);
  count_launch();
  sel_greedy_kernel<<<1, 1024, sizeof(SelJob) * SEL_MAX_CAND, stream>>>(*d, ku, n_cand, cand,
                                                                         slack, budget, flags + 1);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  PASTE_CUDA_CHECK(cudaMemcpyAsync(h_flags, flags, sizeof(h_flags), cudaMemcpyDeviceToHost, stream));
  PASTE_CUDA_CHECK(cudaStreamSynchronize(stream));
  if (h_flags[0]) {
    set_error("jobs need cost >= 1, a non-zero duration and a non-NaN utility");
    return PASTE_ERR_INVALID;
  }
  if (h_flags[1])  // more than SEL_MAX_CAND tied candidates: the general path
    return select_general(d, slack, budget, cap64, ku, gen, gen_end, stream);
  return PASTE_OK;
}

extern "C" int64_t paste_select_scratch_bytes(int64_t n_jobs) {
  return fast_bytes(n_jobs) + general_bytes(n_jobs);
}

// ---------------------------------------------------------------------------
// Stage-2 preemption victim (scheduling.py:571-578): the running speculative
// job minimising (U, -id).  One CTA sweeps the jobs and reduces.
// ---------------------------------------------------------------------------
namespace paste {

// (U, -id, index): min() returns the first of equal keys
__device__ __forceinline__ bool victim_less(uint64_t ka, uint64_t ia, int32_t xa, uint64_t kb,
                                            uint64_t ib, int32_t xb) {
  if (ka != kb) return ka < kb;
  if (ia != ib) return ia < ib;
  return xa < xb;
}

__global__ void __launch_bounds__(1024) victim_kernel(paste_select_desc D, int32_t* out_idx,
                                                      int* bad) {
  __shared__ uint64_t sk[1024], si[1024];
  __shared__ int32_t sx[1024];
  uint64_t bk = ~0ull, bi = ~0ull;
  int32_t bx = -1;
  for (int64_t i = threadIdx.x; i < D.n_jobs; i += blockDim.x) {
    const double p = D.p[i], c = (double)D.cost[i], d = D.duration[i];
    const double u = __ddiv_rn(__dmul_rn(p, D.benefit[i]), __dmul_rn(c, d));
    if (d == 0.0 || D.cost[i] == 0 || u != u) atomicOr(bad, 1);
    const uint64_t ku = ~desc_key(u);                                   // ascending U
    const uint64_t ki = ~((uint64_t)D.id[i] ^ 0x8000000000000000ull);  // larger id first
    if (bx < 0 || victim_less(ku, ki, (int32_t)i, bk, bi, bx)) {
      bk = ku;
      bi = ki;
      bx = (int32_t)i;
    }
  }
  sk[threadIdx.x] = bk;
  si[threadIdx.x] = bi;
  sx[threadIdx.x] = bx;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      const int o = threadIdx.x + off;
      if (sx[o] >= 0 && (sx[threadIdx.x] < 0 || victim_less(sk[o], si[o], sx[o], sk[threadIdx.x],
                                                            si[threadIdx.x], sx[threadIdx.x]))) {
        sk[threadIdx.x] = sk[o];
        si[threadIdx.x] = si[o];
        sx[threadIdx.x] = sx[o];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out_idx = sx[0];
}

}  // namespace paste

extern "C" int paste_select_victim(const paste_select_desc* d, int32_t* out_idx, void* scratch,
                                   void* stream_) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr && out_idx != nullptr && scratch != nullptr, "null argument");
  cudaStream_t stream = (cudaStream_t)stream_;
  int* bad = static_cast<int*>(scratch);
  PASTE_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), stream));
  victim_kernel<<<1, 1024, 0, stream>>>(*d, out_idx, bad);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  int h_bad = 0;
  PASTE_CUDA_CHECK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, stream));
  PASTE_CUDA_CHECK(cudaStreamSynchronize(stream));
  if (h_bad) {
    set_error("jobs need a non-zero cost * duration and a non-NaN utility");
    return PASTE_ERR_INVALID;
  }
  return PASTE_OK;
}
