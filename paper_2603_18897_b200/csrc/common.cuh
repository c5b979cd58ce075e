// Shared device helpers for libpaste (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "paste.h"

namespace paste {

// ---------------------------------------------------------------------------
// error plumbing (thread-local last error, launch counting)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
void count_launch(int n = 1);
void reset_launches();

#define PASTE_CUDA_CHECK(expr)                                                   \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::paste::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,              \
                         cudaGetErrorString(_e));                                \
      return PASTE_ERR_CUDA;                                                     \
    }                                                                            \
  } while (0)

#define PASTE_REQUIRE(cond, ...)                                                 \
  do {                                                                           \
    if (!(cond)) {                                                               \
      ::paste::set_error(__VA_ARGS__);                                           \
      return PASTE_ERR_INVALID;                                                  \
    }                                                                            \
  } while (0)

// ---------------------------------------------------------------------------
// tape access
// ---------------------------------------------------------------------------
struct Node {
  uint32_t type_flags;  // byte0 type, byte1 flags
  int32_t key;
  uint32_t a, b;
  __device__ __forceinline__ int type() const { return type_flags & 0xff; }
  __device__ __forceinline__ int flags() const { return (type_flags >> 8) & 0xff; }
  __device__ __forceinline__ uint32_t size() const { return type() >= PASTE_T_LIST ? b : 1u; }
};

__device__ __forceinline__ Node load_node(const paste_tape_node* nodes, int64_t i) {
  uint4 v = __ldg(reinterpret_cast<const uint4*>(nodes) + i);
  Node n;
  n.type_flags = v.x;
  n.key = (int32_t)v.y;
  n.a = v.z;
  n.b = v.w;
  return n;
}

// Walk one path step from node `cur` (relative to node_base).  Returns the
// child node index, or -1 when the step does not resolve (mappings.py:143-153:
// int step needs a list and 0 <= step < len; key step needs a dict holding it).
__device__ __forceinline__ int64_t step_child(const paste_tape_node* nodes, int64_t base,
                                              int64_t cur, int32_t kind, int32_t value) {
  Node nd = load_node(nodes, base + cur);
  int64_t child = cur + 1;
  if (kind == 0) {
    if (nd.type() != PASTE_T_DICT) return -1;
    for (uint32_t c = 0; c < nd.a; ++c) {
      Node cn = load_node(nodes, base + child);
      if (cn.key == value) return child;
      child += cn.size();
    }
    return -1;
  }
  if (nd.type() != PASTE_T_LIST || value < 0 || (uint32_t)value >= nd.a) return -1;
  for (int32_t c = 0; c < value; ++c) child += load_node(nodes, base + child).size();
  return child;
}

// Walk `bd`'s path (plus the fallback index) from the root of event `ev`.
__device__ __forceinline__ int64_t walk_binding(const paste_windows& win, const int32_t* steps,
                                                const paste_binding& bd, int64_t nb, int fails) {
  int64_t cur = 0;
  const int2* st = reinterpret_cast<const int2*>(steps);
  for (int s = 0; s < bd.step_cnt && cur >= 0; ++s) {
    const int2 k = __ldg(st + bd.step_off + s);
    cur = step_child(win.nodes, nb, cur, k.x, k.y);
  }
  if (bd.kind == PASTE_X_FALLBACK) {
    if (cur >= 0)
      cur = bd.start_index < 0 ? -1 : step_child(win.nodes, nb, cur, 1, bd.start_index + fails);
    for (int s = 0; s < bd.suf_cnt && cur >= 0; ++s) {
      const int2 k = __ldg(st + bd.suf_off + s);
      cur = step_child(win.nodes, nb, cur, k.x, k.y);
    }
  } else if (bd.kind == PASTE_X_FORMAT && cur >= 0) {
    // _leaf_str: only str / number leaves fill the hole (mappings.py:197-204)
    const int t = load_node(win.nodes, nb + cur).type();
    if (t != PASTE_T_STR && t != PASTE_T_INT && t != PASTE_T_FLOAT) cur = -1;
  }
  return cur;
}

// ---------------------------------------------------------------------------
// window-ring / output-record addressing (session-major or slot-major)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t ring_at(const paste_windows& w, int64_t sess, int slot) {
  if (w.stream_end) return w.stream_end[sess] - w.count[sess] + slot;  // stream mode (count <= W)
  return w.slot_major ? (int64_t)slot * w.n_sessions + sess : sess * w.capacity + slot;
}
__host__ __device__ __forceinline__ int64_t out_at(const paste_predict_out& o, int64_t n,
                                                   int64_t sess, int i) {
  return o.slot_major ? (int64_t)i * n + sess : sess * o.max_candidates + i;
}
__host__ __device__ __forceinline__ int64_t arg_at(const paste_predict_out& o, int64_t n,
                                                   int64_t sess, int i, int b) {
  return o.slot_major ? ((int64_t)i * o.max_bindings + b) * n + sess
                      : (sess * o.max_candidates + i) * o.max_bindings + b;
}

// ---------------------------------------------------------------------------
// byte-range helpers: 32-bit word loads (2 aligned loads + funnel shift) so a
// ~20-byte comparison is ~10 loads in flight instead of ~40 dependent byte
// loads.  Loads never touch a 4-byte word that holds no byte of the range, so
// they stay inside the allocation.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_part(const uint8_t* p, int r) {  // r in 1..4 bytes
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  const uint32_t sh = (uint32_t)(a & 3);
  const uint32_t lo = __ldg(w);
  const uint32_t hi = (sh + r > 4) ? __ldg(w + 1) : 0u;
  const uint32_t v = __funnelshift_r(lo, hi, sh * 8);
  return r >= 4 ? v : (v & ((1u << (8 * r)) - 1u));
}

// r in 1..8 bytes at p, from aligned 8-byte words that each hold a byte of
// the range (device allocations are at least 8-byte granular)
__device__ __forceinline__ uint64_t ld_part8(const uint8_t* p, int r) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint64_t* w = reinterpret_cast<const uint64_t*>(a & ~uintptr_t(7));
  const uint32_t o = (uint32_t)(a & 7);
  uint64_t v = __ldg(w) >> (8 * o);
  if (o + r > 8) v |= __ldg(w + 1) << (64 - 8 * o);  // o > 0 here
  return r >= 8 ? v : (v & ((1ull << (8 * r)) - 1ull));
}

__device__ __forceinline__ bool bytes_eq(const uint8_t* a, const uint8_t* b, int64_t n) {
  for (int64_t k = 0; k < n; k += 8) {
    const int r = n - k < 8 ? (int)(n - k) : 8;
    if (ld_part8(a + k, r) != ld_part8(b + k, r)) return false;
  }
  return true;
}

// ---------------------------------------------------------------------------
// narrow record streams (paste_compact_desc, element widths per format)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cf_hdr(const paste_compact_desc& C, int64_t s, int np, int nq) {
  if (C.format & PASTE_CF_HDR8) static_cast<uint8_t*>(C.hdr)[s] = (uint8_t)(np | (nq << 4));
  else static_cast<uint16_t*>(C.hdr)[s] = (uint16_t)(np | (nq << 8));
}
__device__ __forceinline__ void cf_pred(const paste_compact_desc& C, int64_t i, int pid, int comp) {
  if (C.format & PASTE_CF_PRED8) static_cast<uint8_t*>(C.pred)[i] = (uint8_t)(pid | (comp << 6));
  else static_cast<uint16_t*>(C.pred)[i] = (uint16_t)(pid | (comp << 14));
}
// argument ref r (event << 32 | node, < 0 = unresolved) of session s; false
// when the ref does not fit the chosen form (written as unresolved)
__device__ __forceinline__ bool cf_arg(const paste_compact_desc& C, int64_t i, int64_t r,
                                       int64_t n, int64_t s) {
  const bool a16 = (C.format & PASTE_CF_ARG16) != 0;
  uint32_t w = a16 ? 0xffffu : 0xffffffffu;
  bool ok = true;
  if (r >= 0) {
    // event ids are int32 (the window rings), so a 32-bit division suffices
    const int64_t ev = r >> 32, node = r & 0xffffffffll;
    const int64_t region = n < (1ll << 31) ? (int64_t)((uint32_t)ev / (uint32_t)n) : ev / n;
    if (ev - region * n == s && region < 31 && node < (a16 ? (1ll << 11) : (1ll << 27)))
      w = a16 ? (((uint32_t)region << 11) | (uint32_t)node) : (((uint32_t)region << 27) | (uint32_t)node);
    else
      ok = false;
  }
  if (a16) static_cast<uint16_t*>(C.arg)[i] = (uint16_t)w;
  else static_cast<uint32_t*>(C.arg)[i] = w;
  return ok;
}

// ---------------------------------------------------------------------------
// Decoupled look-back over 4 running counters (stream compaction offsets).
// Tile state: one 128-byte line per tile: flag (0 none, 1 aggregate, 2
// inclusive prefix), the 4 tile aggregates, the 4 inclusive prefixes.  Call
// with a whole warp; lane L checks predecessors w - 4L - j (j < 4), so the
// inclusive-prefix frontier advances 128 tiles per L2 round trip.
// ---------------------------------------------------------------------------
constexpr int LB_STRIDE = 16;  // u64 per tile record

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void tile_lookback(uint64_t* tile_state, int64_t tile,
                                              const uint64_t agg[4], uint64_t excl[4], int lane) {
  uint64_t* rec = tile_state + LB_STRIDE * tile;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) st_relaxed(rec + (tile == 0 ? 5 : 1) + k, agg[k]);
    __threadfence();
    st_relaxed(rec, tile == 0 ? 2 : 1);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) excl[k] = 0;
  for (int64_t w = tile - 1; w >= 0; w -= 128) {
    uint64_t fl[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t idx = w - 4 * lane - j;
      fl[j] = 2;  // before tile 0: an inclusive prefix of 0
      if (idx >= 0)
        do {
          fl[j] = ld_relaxed(tile_state + LB_STRIDE * idx);
        } while (fl[j] == 0);
    }
    __threadfence();
    int first = 4;  // this lane's first predecessor holding a prefix
#pragma unroll
    for (int j = 3; j >= 0; --j)
      if (fl[j] == 2) first = j;
    const unsigned pre = __ballot_sync(0xffffffffu, first < 4);
    const int stop = pre ? __ffs(pre) - 1 : 32;
    uint64_t val[4] = {0, 0, 0, 0};
    if (lane <= stop) {
      const int jmax = lane < stop ? 3 : first;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t idx = w - 4 * lane - j;
        if (j > jmax || idx < 0) continue;
        const uint64_t* r = tile_state + LB_STRIDE * idx + (fl[j] == 2 ? 5 : 1);
#pragma unroll
        for (int k = 0; k < 4; ++k) val[k] += ld_relaxed(r + k);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) val[k] += __shfl_xor_sync(0xffffffffu, val[k], o);
      excl[k] += val[k];
    }
    if (pre) break;
  }
  if (lane == 0 && tile > 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) st_relaxed(rec + 5 + k, excl[k] + agg[k]);
    __threadfence();
    st_relaxed(rec, 2);
  }
}

// K4 fast path (predict_fast.cu); false = not eligible, use the generic kernel
bool predict_fast_dispatch(const paste_pool_desc* pool, const paste_windows* win,
                           const paste_admit_desc* adm, const paste_predict_out* out, int G,
                           cudaStream_t stream);

}  // namespace paste
