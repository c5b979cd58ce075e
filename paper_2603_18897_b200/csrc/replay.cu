// C2 replay: score_accuracy (prediction.py:133-169) as three launches.
//
//   1. replay_windows_kernel: each scored call's window (the `call_len` events
//      before it in the event stream) is gathered into a slot-major ring, the
//      layout K4 reads;
//   2. K4 (paste_predict_batch) predicts every window;
//   3. replay_score_kernel: one thread per call tallies top1 / top3 and the
//      hit check -- a FULL candidate of the call's tool whose arguments
//      canonically equal the call's (canonical_arg_hash, events.py:95-118).
//
// Canonical equality of two argument dicts = equal key sets (key-set ids the
// host interns from the NFC key strings) and, per key, equal canonical values.
// For scalars canonical_form maps an integral float to an int, keeps bool
// apart from int and NFC-normalises strings; json.dumps is injective on the
// result, so "equal canonical JSON" is "same tape type class and same
// canonical bytes" (NaN == NaN here, unlike values_equal).  Values that need
// more -- containers on both sides, non-ASCII FormatTemplate text, lone
// surrogates (json.dumps(...).encode raises on them) -- make the call
// "unsure"; the host re-checks those calls with the reference semantics.
#include "common.cuh"

namespace paste {

__global__ void replay_windows_kernel(const paste_replay_desc D, int32_t* __restrict__ tok,
                                      int32_t* __restrict__ evt, int64_t* __restrict__ count) {
  const int64_t n = D.n_calls;
  const int W = D.capacity;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * W;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int slot = (int)(t / n);
    const int64_t c = t - (int64_t)slot * n;
    const int len = D.call_len[c];
    int32_t tk = -1, ev = -1;
    if (slot < len) {
      const int64_t g = D.call_pos[c] - len + slot;
      tk = D.ev_tok[g];
      ev = D.ev_evt[g];
    }
    tok[t] = tk;
    evt[t] = ev;
    if (slot == 0) count[c] = len;
  }
}

__device__ __forceinline__ bool has_surrogate(const uint8_t* b, int64_t n) {
  for (int64_t k = 0; k + 1 < n; ++k)
    if (b[k] == 0xED && b[k + 1] >= 0xA0) return true;
  return false;
}

// Canonical bytes of a scalar node: NFC variant for strings.
__device__ __forceinline__ const uint8_t* canon_bytes(const paste_replay_desc& D, const Node& nd,
                                                      int64_t byte_base, int64_t* len) {
  const uint8_t* b = D.bytes + byte_base + nd.a;
  *len = nd.b;
  if (nd.type() == PASTE_T_STR && (nd.flags() & PASTE_F_NFC)) {
    const uint8_t* x = b + nd.b;
    *len = (int64_t)x[0] | ((int64_t)x[1] << 8) | ((int64_t)x[2] << 16) | ((int64_t)x[3] << 24);
    b = x + 4;
  }
  return b;
}

__device__ __forceinline__ bool py_space_ascii(uint8_t c) {
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 28 && c <= 31);
}

enum { CMP_NE = 0, CMP_EQ = 1, CMP_UNSURE = 2 };

// Predicted value of binding `bind` (node `pref` = event << 32 | node) vs the
// actual argument node `an` of payload `aev`.
__device__ int compare_binding(const paste_replay_desc& D, int bind, int kind, int64_t pref,
                               int32_t aev, int64_t an) {
  const int32_t pev = (int32_t)(pref >> 32);
  const paste_event_ref pr = D.refs[pev], ar = D.refs[aev];
  const Node pn = load_node(D.nodes, pr.node_base + (pref & 0xFFFFFFFF));
  const Node a = load_node(D.nodes, ar.node_base + an);
  const int at = a.type();
  int64_t al;
  const uint8_t* ab = at < PASTE_T_LIST ? canon_bytes(D, a, ar.byte_base, &al) : nullptr;
  if (kind != PASTE_X_FORMAT) {
    const int pt = pn.type();
    if (pt >= PASTE_T_LIST || at >= PASTE_T_LIST) return pt == at ? CMP_UNSURE : CMP_NE;
    if (pt != at) return CMP_NE;
    if (pt <= PASTE_T_TRUE) return CMP_EQ;
    int64_t pl;
    const uint8_t* pb = canon_bytes(D, pn, pr.byte_base, &pl);
    if (pt == PASTE_T_STR && (has_surrogate(pb, pl) || has_surrogate(ab, al))) return CMP_UNSURE;
    if (pl != al) return CMP_NE;
    for (int64_t k = 0; k < pl; ++k)
      if (pb[k] != ab[k]) return CMP_NE;
    return CMP_EQ;
  }
  // FormatTemplate: prefix + norm(leaf_str(leaf)) + suffix (mappings.py:197-223)
  if (at != PASTE_T_STR) return CMP_NE;
  const uint8_t* tb = D.bytes + pr.byte_base + pn.a;  // leaf_str: raw text / number text
  int64_t lo = 0, hi = pn.b;
  const int* f = D.fmt + 5 * bind;
  const uint8_t* pre = D.fmt_bytes + f[0];
  const uint8_t* suf = D.fmt_bytes + f[2];
  const int pl = f[1], sl = f[3], norm = f[4];
  bool ascii = true;
  for (int64_t k = 0; k < hi; ++k) ascii &= tb[k] < 0x80;
  for (int k = 0; k < pl; ++k) ascii &= pre[k] < 0x80;
  for (int k = 0; k < sl; ++k) ascii &= suf[k] < 0x80;
  for (int64_t k = 0; k < al; ++k) ascii &= ab[k] < 0x80;
  if (!ascii) return CMP_UNSURE;
  if (norm == 1) {  // str.strip()
    while (lo < hi && py_space_ascii(tb[lo])) ++lo;
    while (hi > lo && py_space_ascii(tb[hi - 1])) --hi;
  }
  if ((int64_t)pl + (hi - lo) + sl != al) return CMP_NE;
  for (int k = 0; k < pl; ++k)
    if (pre[k] != ab[k]) return CMP_NE;
  for (int64_t k = lo; k < hi; ++k) {
    uint8_t c = tb[k];
    if (norm == 2 && c >= 'A' && c <= 'Z') c += 32;  // str.lower()
    if (c != ab[pl + (k - lo)]) return CMP_NE;
  }
  for (int k = 0; k < sl; ++k)
    if (suf[k] != ab[pl + (hi - lo) + k]) return CMP_NE;
  return CMP_EQ;
}

__device__ __forceinline__ int64_t lookup_key(const paste_tape_node* nodes, int64_t base,
                                              int32_t key) {
  return step_child(nodes, base, 0, 0, key);
}

__global__ void __launch_bounds__(256) replay_score_kernel(const paste_pool_desc pool,
                                                           const paste_replay_desc D,
                                                           const paste_predict_out out) {
  unsigned long long c1 = 0, c3 = 0, ch = 0, cu = 0;
  const int64_t n = D.n_calls;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    int np = out.n_pred[c];
    const int lim = D.cand_limit;
    np = lim >= 0 ? (np < lim ? np : lim) : (np + lim > 0 ? np + lim : 0);
    const int32_t tool = D.call_tool[c];
    bool top1 = false, top3 = false, hit = false, unsure = false;
    const int32_t cks = D.call_keyset[c];
    const int32_t aev = D.call_args[c];
    for (int i = 0; i < np && !hit; ++i) {
      const int64_t o = out_at(out, n, c, i);
      const int32_t pid = out.pred_pat[o];
      const paste_pattern pat = pool.patterns[pid];
      const bool same = pat.target_tool == tool;
      if (i == 0) top1 = same;
      if (i < 3) top3 |= same;
      if (!same || out.pred_comp[o] != PASTE_C_FULL) continue;
      const int32_t pks = D.pat_keyset[pid];
      if (cks == -2) continue;                       // args not a dict: never equal
      if (pks < 0 || cks < 0) { unsure = true; continue; }
      if (pks != cks) continue;
      const int nb = (pat.flags & PASTE_PF_HAS_MAPPING) ? pat.n_bind : 0;
      int verdict = CMP_EQ;
      for (int b = 0; b < nb && verdict != CMP_NE; ++b) {
        const int bind = pat.bind_off + b;
        const int64_t pref = out.pred_arg[arg_at(out, n, c, i, b)];
        const int64_t an = lookup_key(D.nodes, D.refs[aev].node_base, D.bind_key[bind]);
        if (pref < 0 || an < 0) { verdict = CMP_UNSURE; continue; }  // FULL + equal key sets
        const int r = compare_binding(D, bind, pool.bindings[bind].kind, pref, aev, an);
        if (r == CMP_NE) verdict = CMP_NE;
        else if (r == CMP_UNSURE) verdict = CMP_UNSURE;
      }
      if (verdict == CMP_EQ) hit = true;
      else if (verdict == CMP_UNSURE) unsure = true;
    }
    if (hit) unsure = false;  // (the loop stops at a hit, after top1/top3 are settled)
    D.unsure[c] = unsure;
    c1 += top1;
    c3 += top3;
    ch += hit;
    cu += unsure;
  }
  // block reduction then one atomic per counter per block
  __shared__ unsigned long long red[4][8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int off = 16; off; off >>= 1) {
    c1 += __shfl_down_sync(0xffffffffu, c1, off);
    c3 += __shfl_down_sync(0xffffffffu, c3, off);
    ch += __shfl_down_sync(0xffffffffu, ch, off);
    cu += __shfl_down_sync(0xffffffffu, cu, off);
  }
  if (lane == 0) {
    red[0][wid] = c1;
    red[1][wid] = c3;
    red[2][wid] = ch;
    red[3][wid] = cu;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    unsigned long long s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[threadIdx.x][w];
    if (s) atomicAdd(reinterpret_cast<unsigned long long*>(D.tallies) + threadIdx.x, s);
  }
}

}  // namespace paste

using namespace paste;

extern "C" int64_t paste_replay_scratch_bytes(int64_t n_calls, int32_t capacity) {
  if (n_calls < 0 || capacity < 1) return -1;
  const int64_t ring = ((n_calls * capacity * 4 + 255) / 256) * 256;
  return 2 * ring + ((n_calls * 8 + 255) / 256) * 256;
}

extern "C" int paste_replay_score(const paste_pool_desc* pool, const paste_replay_desc* d,
                                  paste_predict_out* out, void* scratch, void* stream) {
  reset_launches();
  PASTE_REQUIRE(pool && d && out, "null descriptor");
  PASTE_REQUIRE(d->capacity >= 1, "window capacity must be >= 1");
  if (d->n_calls == 0) return PASTE_OK;
  PASTE_REQUIRE(scratch != nullptr, "null scratch");
  const cudaStream_t st = (cudaStream_t)stream;
  const int64_t ring = ((d->n_calls * d->capacity * 4 + 255) / 256) * 256;
  uint8_t* s = static_cast<uint8_t*>(scratch);
  int32_t* tok = reinterpret_cast<int32_t*>(s);
  int32_t* evt = reinterpret_cast<int32_t*>(s + ring);
  int64_t* count = reinterpret_cast<int64_t*>(s + 2 * ring);
  const int threads = 256;
  int64_t blocks = (d->n_calls * d->capacity + threads - 1) / threads;
  if (blocks > 148 * 32) blocks = 148 * 32;
  replay_windows_kernel<<<(unsigned)blocks, threads, 0, st>>>(*d, tok, evt, count);
  PASTE_CUDA_CHECK(cudaGetLastError());

  paste_windows win{};
  win.n_sessions = d->n_calls;
  win.capacity = d->capacity;
  win.slot_major = 1;
  win.tok = tok;
  win.evt = evt;
  win.count = count;
  win.nodes = d->nodes;
  win.bytes = d->bytes;
  win.refs = const_cast<paste_event_ref*>(d->refs);  // read-only: no observe step
  paste_admit_desc adm{};
  const int rc = paste_predict_batch(pool, &win, &adm, out, stream);
  if (rc != PASTE_OK) return rc;

  blocks = (d->n_calls + threads - 1) / threads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  replay_score_kernel<<<(unsigned)blocks, threads, 0, st>>>(*pool, *d, *out);
  PASTE_CUDA_CHECK(cudaGetLastError());
  count_launch(2);  // + the K4 launches counted by paste_predict_batch
  return PASTE_OK;
}
