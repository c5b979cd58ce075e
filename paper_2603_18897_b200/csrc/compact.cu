// Record compaction for the live path: fixed K-slot predict records ->
// narrow CSR streams sized by what each session actually produced, so the
// device->host copy of a live step moves ~24 B/session instead of the fixed
// 204 B (K = 8).
//
// Single pass with a decoupled look-back scan: CTAs claim 128-session tiles
// through a ticket counter (tiles are therefore taken in order and every
// predecessor is running or done), publish their tile aggregates, look back
// for the exclusive prefix, publish the inclusive prefix and scatter.
//
// Streams (all in session order):
//   hdr[n]      u16  n_pred | n_act << 8  (u8, 4 + 4 bits, with PASTE_CF_HDR8)
//   pred[P]     u16  pattern id | completeness << 14  (u8, 6 + 2 bits: PRED8)
//   arg[A]      u32  argument refs of MAPPED predictions only (n_bind each):
//                    region << 27 | node, where the source event is
//                    region * n + session (the live table's event ids); a
//                    ref outside that form is counted in totals[3] and
//                    written as all-ones (the caller re-fetches full records)
//                    (u16, region << 11 | node, with PASTE_CF_ARG16)
//   act[Q]      u8   prediction slot | level << 5
// The expected utility of an action is p(pattern) * benefit(tool), one
// IEEE multiply the host redoes exactly on decode, so it is not shipped.
#include "common.cuh"

namespace paste {

constexpr int KT_T = 128;  // sessions per tile / threads per CTA
constexpr uint64_t ST_AGG = 1ull << 62, ST_PRE = 2ull << 62, ST_MASK = 3ull << 62;

__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(KT_T) compact_kernel(const paste_predict_out O, int64_t n,
                                                       const paste_pattern* patterns,
                                                       paste_compact_desc C, uint64_t* ticket,
                                                       uint64_t* tile_state) {
  __shared__ int64_t s_tile;
  __shared__ uint64_t s_sum[3][KT_T];
  __shared__ uint64_t s_excl[3];
  if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(ticket), 1ull);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t s = tile * KT_T + threadIdx.x;
  const int K = O.max_candidates, B = O.max_bindings;
  const int64_t ostride = O.slot_major ? n : 1;
  const int64_t obase = O.slot_major ? s : s * K;
  const int64_t abase = O.slot_major ? s : s * K * B;
  int np = 0, na = 0, nq = 0;
  if (s < n) {
    np = O.n_pred[s];
    nq = O.n_act ? O.n_act[s] : 0;
    for (int i = 0; i < np; ++i) {
      const int pid = O.pred_pat[obase + i * ostride];
      const paste_pattern pt = patterns[pid];
      if (pt.flags & PASTE_PF_HAS_MAPPING) na += pt.n_bind;
    }
  }
  // block-wide inclusive scans of (np, na, nq)
  uint64_t v[3] = {(uint64_t)np, (uint64_t)na, (uint64_t)nq};
  for (int c = 0; c < 3; ++c) s_sum[c][threadIdx.x] = v[c];
  __syncthreads();
  for (int off = 1; off < KT_T; off <<= 1) {
    uint64_t add[3];
    for (int c = 0; c < 3; ++c) add[c] = threadIdx.x >= off ? s_sum[c][threadIdx.x - off] : 0;
    __syncthreads();
    for (int c = 0; c < 3; ++c) s_sum[c][threadIdx.x] += add[c];
    __syncthreads();
  }
  // look-back (one thread per counter)
  if (threadIdx.x < 3) {
    const int c = threadIdx.x;
    const uint64_t agg = s_sum[c][KT_T - 1];
    uint64_t* st = tile_state + 3 * tile + c;
    if (tile == 0) {
      st_release(st, ST_PRE | agg);
      s_excl[c] = 0;
    } else {
      st_release(st, ST_AGG | agg);
      uint64_t excl = 0;
      for (int64_t j = tile - 1; j >= 0; --j) {
        uint64_t w;
        do {
          w = ld_acquire(tile_state + 3 * j + c);
        } while ((w & ST_MASK) == 0);
        excl += w & ~ST_MASK;
        if ((w & ST_MASK) == ST_PRE) break;
      }
      st_release(st, ST_PRE | (excl + agg));
      s_excl[c] = excl;
    }
  }
  __syncthreads();
  if (s < n) {
    uint64_t p0 = s_excl[0] + s_sum[0][threadIdx.x] - np;
    uint64_t a0 = s_excl[1] + s_sum[1][threadIdx.x] - na;
    uint64_t q0 = s_excl[2] + s_sum[2][threadIdx.x] - nq;
    cf_hdr(C, s, np, nq);
    unsigned long long wide = 0;
    for (int i = 0; i < np; ++i) {
      const int64_t o = obase + i * ostride;
      const int pid = O.pred_pat[o];
      cf_pred(C, p0 + i, pid, (int)O.pred_comp[o]);
      const paste_pattern pt = patterns[pid];
      if (pt.flags & PASTE_PF_HAS_MAPPING)
        for (int b = 0; b < pt.n_bind; ++b)
          wide += !cf_arg(C, a0++, O.pred_arg[abase + (int64_t)(i * B + b) * ostride], n, s);
    }
    for (int j = 0; j < nq; ++j) {
      const int64_t o = obase + j * ostride;
      C.act[q0 + j] = (uint8_t)(O.act_pred[o] | (O.act_level[o] << 5));
    }
    if (wide) atomicAdd(reinterpret_cast<unsigned long long*>(C.totals + 3), wide);
    if (O.struct_err && O.struct_err[s])
      atomicAdd(reinterpret_cast<unsigned long long*>(C.totals + 4),
                (unsigned long long)O.struct_err[s]);
  }
  if (s == n - 1) {
    C.totals[0] = s_excl[0] + s_sum[0][threadIdx.x];
    C.totals[1] = s_excl[1] + s_sum[1][threadIdx.x];
    C.totals[2] = s_excl[2] + s_sum[2][threadIdx.x];
  }
}

}  // namespace paste

using namespace paste;

extern "C" int64_t paste_compact_scratch_bytes(int64_t n_sessions) {
  const int64_t tiles = (n_sessions + KT_T - 1) / KT_T;
  return 8 * (3 * tiles + 1);
}

extern "C" int paste_compact_records(const paste_predict_out* out, int64_t n_sessions,
                                     const paste_pool_desc* pool, paste_compact_desc* c,
                                     void* scratch, void* stream_) {
  reset_launches();
  PASTE_REQUIRE(out && pool && c && scratch, "null argument");
  PASTE_REQUIRE(out->max_candidates <= 31 && pool->n_patterns <= (1 << 14),
                "compaction needs max_candidates <= 31 and at most 16384 patterns");
  PASTE_REQUIRE(!(c->format & PASTE_CF_HDR8) || out->max_candidates <= 15,
                "PASTE_CF_HDR8 needs max_candidates <= 15");
  PASTE_REQUIRE(!(c->format & PASTE_CF_PRED8) || pool->n_patterns <= 64,
                "PASTE_CF_PRED8 needs at most 64 patterns");
  cudaStream_t stream = (cudaStream_t)stream_;
  const int64_t tiles = (n_sessions + KT_T - 1) / KT_T;
  PASTE_CUDA_CHECK(cudaMemsetAsync(scratch, 0, paste_compact_scratch_bytes(n_sessions), stream));
  PASTE_CUDA_CHECK(cudaMemsetAsync(c->totals, 0, 5 * sizeof(int64_t), stream));
  if (n_sessions == 0) return PASTE_OK;
  uint64_t* ticket = static_cast<uint64_t*>(scratch);
  compact_kernel<<<(unsigned)tiles, KT_T, 0, stream>>>(*out, n_sessions, pool->patterns, *c, ticket,
                                                       ticket + 1);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
