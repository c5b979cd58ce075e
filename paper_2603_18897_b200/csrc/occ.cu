// Phase II occurrence collection (_collect_occurrences, mining.py:215-227,
// with mine()'s filter to followed occurrences of the target, :277-279) for
// every mapping candidate in one pass over the flagged token stream.
//
// One thread per anchor.  The candidates that can match at anchor a are
// exactly those whose context ends with sig(a) and whose target is the tool
// of the next event, so a (last sig, target tool) bucket table (built on the
// host from the selected candidates) bounds the work per anchor to the
// candidates that share both.  match_at (mining.py:119-156) is evaluated on
// the tokens: the anchored rightmost embedding walks back from a - 1 to
// max(stream start, a - k + 1) greedily (greedy from the right is the
// rightmost embedding), the contiguous suffix compares the slice ending at
// a.  The stream boundary is the SEG_START bit of the first token of every
// session stream: a position p < a is in a's stream iff no token in
// (p, a] carries it.
//
// Slots are claimed with one atomic per emission inside the candidate's
// range (the range sizes are the mining tables' follow counts, so the
// emission is exact); the stream order inside a range is restored by the
// caller with the K1 sort (paste_ingest_order).
#include "common.cuh"

namespace paste {
namespace {

constexpr int OCC_T = 256;
constexpr int32_t SEG_FLAG = (int32_t)0x80000000;

__global__ void __launch_bounds__(OCC_T) occurrences_kernel(const paste_occ_desc d) {
  const int64_t n = d.n_tokens;
  const int64_t stride = (int64_t)gridDim.x * OCC_T;
  unsigned long long over = 0;
  for (int64_t a = (int64_t)blockIdx.x * OCC_T + threadIdx.x; a + 1 < n; a += stride) {
    const int32_t t1 = __ldg(d.tok + a + 1);
    if (t1 < 0) continue;  // the next event opens another stream
    const int32_t s = __ldg(d.tok + a) & 0x7fffffff;
    const int64_t b = (int64_t)s * d.n_tools + (t1 >> 1);
    const int32_t i0 = __ldg(d.bucket_off + b), i1 = __ldg(d.bucket_off + b + 1);
    for (int32_t i = i0; i < i1; ++i) {
      const int32_t c = __ldg(d.bucket + i);
      const int L = __ldg(d.ctx_len + c);
      const int32_t* ctx = d.ctx + (int64_t)c * d.kmax;
      int32_t pk[16];
      pk[L - 1] = (int32_t)a;
      bool ok;
      if (d.relation == 1) {  // contiguous suffix: the slice stream[a - L + 1 .. a]
        ok = a - (L - 1) >= 0;
        for (int j = L - 2; ok && j >= 0; --j) {
          const int64_t p = a - (L - 1 - j);
          const int32_t tp1 = __ldg(d.tok + p + 1);
          if (tp1 < 0) {  // p + 1 opens a's stream: p is outside it
            ok = false;
            break;
          }
          ok = (__ldg(d.tok + p) & 0x7fffffff) == __ldg(ctx + j);
          pk[j] = (int32_t)p;
        }
      } else {  // anchored: rightmost embedding inside [max(start, a - k + 1), a]
        int j = L - 2;
        int64_t p = a - 1;
        const int64_t lo = a - d.k + 1;
        while (j >= 0 && p >= lo && p >= 0 && __ldg(d.tok + p + 1) >= 0) {
          if ((__ldg(d.tok + p) & 0x7fffffff) == __ldg(ctx + j)) pk[j--] = (int32_t)p;
          --p;
        }
        ok = j < 0;
      }
      if (!ok) continue;
      const int64_t slot = __ldg(d.off + c) +
                           (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(d.cursor + c), 1ull);
      if (slot >= __ldg(d.off + c + 1)) {
        ++over;
        continue;
      }
      d.anchor[slot] = a;
      for (int j = 0; j < L; ++j) d.picked[slot * d.kmax + j] = pk[j];
    }
  }
  if (over) atomicAdd(reinterpret_cast<unsigned long long*>(d.overflow), over);
}

}  // namespace
}  // namespace paste

extern "C" int paste_mine_occurrences(const paste_occ_desc* d, void* stream) {
  using namespace paste;
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null occurrence descriptor");
  PASTE_REQUIRE(d->n_cand >= 0 && d->n_tokens >= 0, "negative sizes");
  PASTE_REQUIRE(d->kmax >= 1 && d->kmax <= 16, "kmax must be in [1, 16]");
  PASTE_REQUIRE(d->relation == 0 || d->relation == 1, "relation must be 0 or 1");
  PASTE_REQUIRE(d->n_tokens < ((int64_t)1 << 31), "picked positions are int32: n_tokens < 2^31");
  if (d->n_cand == 0 || d->n_tokens < 2) return PASTE_OK;
  PASTE_REQUIRE(d->tok && d->ctx && d->ctx_len && d->bucket_off && d->bucket && d->off &&
                    d->cursor && d->anchor && d->picked && d->overflow,
                "null array");
  int64_t blocks = (d->n_tokens + OCC_T - 1) / OCC_T;
  if (blocks > 148 * 16) blocks = 148 * 16;
  occurrences_kernel<<<(unsigned)blocks, OCC_T, 0, (cudaStream_t)stream>>>(*d);
  PASTE_CUDA_CHECK(cudaGetLastError());
  count_launch(1);
  return PASTE_OK;
}
