// Record compaction for the live path: fixed K-slot predict records ->
// narrow CSR streams sized by what each session actually produced, so the
// device->host copy of a live step moves ~24 B/session instead of the fixed
// 204 B (K = 8).
//
// Single pass with a decoupled look-back scan: CTAs claim 128-session tiles
// through a ticket counter (tiles are therefore taken in order and every
// predecessor is running or done), publish their tile aggregates, look back
// for the exclusive prefix with one warp (tile_lookback, common.cuh),
// publish the inclusive prefix and scatter.
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

__global__ void __launch_bounds__(KT_T) compact_kernel(const paste_predict_out O, int64_t n,
                                                       const paste_pattern* patterns,
                                                       paste_compact_desc C, uint64_t* ticket,
                                                       uint64_t* tile_state, int64_t n_tiles) {
  __shared__ int64_t s_tile;
  __shared__ uint64_t s_warp[KT_T / 32][4];
  __shared__ uint64_t s_excl[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(ticket), 1ull);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t s = tile * KT_T + threadIdx.x;
  const int K = O.max_candidates, B = O.max_bindings;
  const int64_t ostride = O.slot_major ? n : 1;
  const int64_t obase = O.slot_major ? s : s * K;
  const int64_t abase = O.slot_major ? s : s * K * B;
  int c[4] = {0, 0, 0, 0};  // predictions, arguments, actions, structural errors
  if (s < n) {
    c[0] = O.n_pred[s];
    c[2] = O.n_act ? O.n_act[s] : 0;
    c[3] = O.struct_err ? O.struct_err[s] : 0;
    for (int i = 0; i < c[0]; ++i) {
      const paste_pattern pt = patterns[O.pred_pat[obase + i * ostride]];
      if (pt.flags & PASTE_PF_HAS_MAPPING) c[1] += pt.n_bind;
    }
  }
  // warp inclusive scans, per-warp sums in shared memory
  uint64_t inc[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint64_t v = (uint64_t)c[k];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint64_t u = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= off) v += u;
    }
    inc[k] = v;
    if (lane == 31) s_warp[warp][k] = v;
  }
  __syncthreads();
  if (warp == 0) {
    uint64_t agg[4], excl[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      agg[k] = 0;
      for (int w = 0; w < KT_T / 32; ++w) agg[k] += s_warp[w][k];
    }
    tile_lookback(tile_state, tile, agg, excl, lane);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) s_excl[k] = excl[k];
      if (tile == n_tiles - 1) {  // the last tile publishes the totals
        C.totals[0] = (int64_t)(excl[0] + agg[0]);
        C.totals[1] = (int64_t)(excl[1] + agg[1]);
        C.totals[2] = (int64_t)(excl[2] + agg[2]);
        C.totals[4] = (int64_t)(excl[3] + agg[3]);
      }
    }
  }
  __syncthreads();
  if (s < n) {
    uint64_t o[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      uint64_t before = 0;
      for (int w = 0; w < warp; ++w) before += s_warp[w][k];
      o[k] = s_excl[k] + before + inc[k] - (uint64_t)c[k];
    }
    cf_hdr(C, s, c[0], c[2]);
    unsigned long long wide = 0;
    uint64_t a0 = o[1];
    for (int i = 0; i < c[0]; ++i) {
      const int64_t oi = obase + i * ostride;
      const int pid = O.pred_pat[oi];
      cf_pred(C, o[0] + i, pid, (int)O.pred_comp[oi]);
      const paste_pattern pt = patterns[pid];
      if (pt.flags & PASTE_PF_HAS_MAPPING)
        for (int b = 0; b < pt.n_bind; ++b)
          wide += !cf_arg(C, a0++, O.pred_arg[abase + (int64_t)(i * B + b) * ostride], n, s);
    }
    for (int j = 0; j < c[2]; ++j) {
      const int64_t oj = obase + j * ostride;
      C.act[o[2] + j] = (uint8_t)(O.act_pred[oj] | (O.act_level[oj] << 5));
    }
    if (wide) atomicAdd(reinterpret_cast<unsigned long long*>(C.totals + 3), wide);
  }
}

}  // namespace paste

using namespace paste;

extern "C" int64_t paste_compact_scratch_bytes(int64_t n_sessions) {
  const int64_t tiles = (n_sessions + KT_T - 1) / KT_T;
  return 8 * (LB_STRIDE * tiles + LB_STRIDE);
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
  if (c->format & PASTE_CF_ENTRY16) {
    set_error("PASTE_CF_ENTRY16 is produced by paste_predict_compact only");
    return PASTE_ERR_UNSUPPORTED;
  }
  cudaStream_t stream = (cudaStream_t)stream_;
  const int64_t tiles = (n_sessions + KT_T - 1) / KT_T;
  PASTE_CUDA_CHECK(cudaMemsetAsync(scratch, 0, paste_compact_scratch_bytes(n_sessions), stream));
  PASTE_CUDA_CHECK(cudaMemsetAsync(c->totals, 0, 5 * sizeof(int64_t), stream));
  if (n_sessions == 0) return PASTE_OK;
  uint64_t* ticket = static_cast<uint64_t*>(scratch);
  compact_kernel<<<(unsigned)tiles, KT_T, 0, stream>>>(*out, n_sessions, pool->patterns, *c, ticket,
                                                       ticket + LB_STRIDE, tiles);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
