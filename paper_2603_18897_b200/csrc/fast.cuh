// Match-table records and the memoised binding walk shared by the K4 fast
// path (predict_fast.cu) and the fused replay (replay.cu).
#pragma once
#include "common.cuh"

namespace paste {

struct MTRecord {  // 32 bytes
  int32_t pid;
  uint32_t src;      // 4-bit source age per binding
  int32_t tool;
  int32_t nb_flags;  // n_bind | flags << 16
  int32_t bind_off;
  int32_t pad;
  double p;
};
static_assert(sizeof(MTRecord) == 32, "MTRecord layout");

// 16-byte header keeps every record 16-byte aligned for the int4 loads
__host__ __device__ inline int64_t mt_stride(int K) { return 16 + 32 * (int64_t)K; }

// ---------------------------------------------------------------------------
// Per-launch walk memo.  With shape-interned payloads many events share one
// node array, and a PathLookup / FormatTemplate walk depends only on (the
// binding, the node array): the CTA memoises those walks in shared memory.
// Entry: valid(1) | binding(16) | node_base(24) | node(23, all-ones = none).
// ---------------------------------------------------------------------------
constexpr int MEMO = 128;
constexpr uint64_t MEMO_NONE = 0x7fffffull;

__device__ __forceinline__ int memo_slot(uint64_t key) {
  return (int)((key * 0x9E3779B97F4A7C15ull) >> 57);  // 7 bits -> 128 slots
}

// Resolve binding `bind` (global index) against source event `ev` at age
// `src_age`; `gt` holds the gathered tokens by age for the failure count.
__device__ __forceinline__ int64_t resolve_fast(const paste_windows& win, const int32_t* steps,
                                                const paste_binding& bd, int bind, int32_t ev,
                                                int src_age, const int32_t* gt, uint64_t* memo) {
  const int64_t nb = win.refs[ev].node_base;
  if (bd.kind == PASTE_X_FALLBACK) {
    int fails = 0;  // FAIL events of fail_tool after the source (mappings.py:185-194)
    for (int a = 0; a < src_age; ++a) {
      const int32_t t = gt[a];
      fails += ((t >> 1) == bd.fail_tool) && ((t & 1) == 0);
    }
    const int64_t cur = walk_binding(win, steps, bd, nb, fails);
    return cur < 0 ? -1 : (((int64_t)ev << 32) | cur);
  }
  const bool cacheable = bind < (1 << 16) && nb < (1ll << 24);
  const uint64_t key = ((uint64_t)bind << 24) | (uint64_t)nb;
  int64_t cur;
  if (cacheable) {
    const int h = memo_slot(key);
    // a lock-free cache shared by the CTA's warps: each entry is one 64-bit
    // word (valid bit, tag, value) read and written with shared-memory
    // atomics, so a reader sees an old or a new entry whole and checks the tag
    unsigned long long* slot = reinterpret_cast<unsigned long long*>(memo + h);
    const uint64_t e = atomicAdd(slot, 0ull);
    if ((e >> 63) && ((e >> 23) & ((1ull << 40) - 1)) == key) {
      const uint64_t v = e & MEMO_NONE;
      cur = v == MEMO_NONE ? -1 : (int64_t)v;
    } else {
      cur = walk_binding(win, steps, bd, nb, 0);
      if (cur < (int64_t)MEMO_NONE)
        atomicExch(slot, (1ull << 63) | (key << 23) | (cur < 0 ? MEMO_NONE : (uint64_t)cur));
    }
  } else {
    cur = walk_binding(win, steps, bd, nb, 0);
  }
  return cur < 0 ? -1 : (((int64_t)ev << 32) | cur);
}

}  // namespace paste
