// K7 phase2_holds: hypothesis hit counts for mapping inference.
//
// Reference: _holds (mappings.py:326-335) evaluates one hypothesis over all
// occurrences: resolve the expression against the occurrence's matched
// context (mappings.py:162-194) and compare with the actual argument
// (values_equal, events.py:125-130).  infer_mapping (mappings.py:276-417)
// tries hypotheses in a fixed order and keeps the first whose hit fraction
// reaches validation_fraction.  Here one thread evaluates one
// (hypothesis, occurrence) pair; the host keeps the enumeration order and
// picks the first passing hypothesis.
//
// Equality:
//   * PathLookup / IndexedFallback: the resolved node must be a scalar of the
//     actual's type class with equal canonical bytes, never NaN (exact);
//   * FormatTemplate: value = prefix + norm(leaf_str(leaf)) + suffix.  When
//     prefix, suffix, leaf text and actual are all ASCII, NFC is the identity
//     and str.strip()/str.lower() act on ASCII only, so the byte comparison is
//     exact; any non-ASCII byte marks the pair "unsure" and the host
//     re-evaluates that hypothesis with Python string semantics.
#include "common.cuh"

namespace paste {

__device__ __forceinline__ bool py_space(uint8_t c) {
  // ASCII characters for which str.isspace() is true
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 28 && c <= 31);
}

__global__ void holds_kernel(const paste_holds_desc D) {
  const int64_t total = D.n_hyp * D.n_occ;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = t / D.n_occ, m = t - h * D.n_occ;
    const paste_binding bd = D.hyp[h];
    bool eq = false, unsure = false;
    // resolve (mappings.py:162-194)
    const int32_t h_lo = D.hist_off[m], h_hi = D.hist_end ? D.hist_end[m] : D.hist_off[m + 1];
    const int32_t ev = D.occ_event[m * D.n_ctx + bd.ctx_pos];
    const paste_event_ref ref = D.refs[ev];
    int64_t cur = 0;
    for (int s = 0; s < bd.step_cnt && cur >= 0; ++s)
      cur = step_child(D.nodes, ref.node_base, cur, D.steps[2 * (bd.step_off + s)],
                       D.steps[2 * (bd.step_off + s) + 1]);
    if (bd.kind == PASTE_X_FALLBACK) {
      int fails = 0;
      const int32_t sp = D.src_pos[m * D.n_ctx + bd.ctx_pos];
      if (sp >= 0)
        for (int32_t q = h_lo + sp + 1; q < h_hi; ++q) {
          const int32_t tk = D.hist_tok[q];
          fails += tk >= 0 && (tk >> 1) == bd.fail_tool && (tk & 1) == 0;
        }
      if (cur >= 0)
        cur = bd.start_index < 0 ? -1
                                 : step_child(D.nodes, ref.node_base, cur, 1, bd.start_index + fails);
      for (int s = 0; s < bd.suf_cnt && cur >= 0; ++s)
        cur = step_child(D.nodes, ref.node_base, cur, D.steps[2 * (bd.suf_off + s)],
                         D.steps[2 * (bd.suf_off + s) + 1]);
    }
    int at;
    bool anan;
    const uint8_t* ab;
    int64_t al;
    if (D.act_event) {  // corpus mode: the actual is a node of the argument tape
      const int32_t an = D.act_node[m];
      at = -1;
      anan = false;
      ab = D.bytes;
      al = 0;
      if (an >= 0) {
        const paste_event_ref aref = D.refs[D.act_event[m]];
        const Node a = load_node(D.nodes, aref.node_base + an);
        if (a.type() < PASTE_T_LIST) {
          at = a.type();
          anan = (a.flags() & PASTE_F_NAN) != 0;
          ab = D.bytes + aref.byte_base + a.a;
          al = a.b;
          if (at == PASTE_T_STR && (a.flags() & PASTE_F_NFC)) {  // canonical: the NFC bytes
            const uint8_t* x = ab + a.b;
            al = (int64_t)x[0] | ((int64_t)x[1] << 8) | ((int64_t)x[2] << 16) |
                 ((int64_t)x[3] << 24);
            ab = x + 4;
          }
        }
      }
    } else {
      at = D.act_type[m];
      anan = D.act_nan[m] != 0;
      ab = D.act_bytes + D.act_off[m];
      al = D.act_off[m + 1] - D.act_off[m];
    }
    if (cur >= 0) {
      const Node nd = load_node(D.nodes, ref.node_base + cur);
      const int nt = nd.type();
      if (bd.kind != PASTE_X_FORMAT) {
        if (nt < PASTE_T_LIST && nt == at && !(nd.flags() & PASTE_F_NAN) && !anan) {
          if (nt <= PASTE_T_TRUE) {
            eq = true;
          } else {
            const uint8_t* b = D.bytes + ref.byte_base + nd.a;
            int64_t len = nd.b;
            if (nt == PASTE_T_STR && (nd.flags() & PASTE_F_NFC)) {
              const uint8_t* x = b + nd.b;
              len = (int64_t)x[0] | ((int64_t)x[1] << 8) | ((int64_t)x[2] << 16) | ((int64_t)x[3] << 24);
              b = x + 4;
            }
            eq = len == al && bytes_eq(b, ab, len);
          }
        }
      } else if ((nt == PASTE_T_STR || nt == PASTE_T_INT || nt == PASTE_T_FLOAT) &&
                 at == PASTE_T_STR) {
        // text = leaf_str(leaf): raw string / canonical number text
        const uint8_t* tb = D.bytes + ref.byte_base + nd.a;
        int64_t lo = 0, hi = nd.b;
        const int norm = D.fmt[5 * h + 4];
        bool ascii = true;
        for (int64_t k = 0; k < hi; ++k) ascii &= tb[k] < 0x80;
        const uint8_t* pre = D.fmt_bytes + D.fmt[5 * h + 0];
        const int pl = D.fmt[5 * h + 1];
        const uint8_t* suf = D.fmt_bytes + D.fmt[5 * h + 2];
        const int sl = D.fmt[5 * h + 3];
        for (int k = 0; k < pl; ++k) ascii &= pre[k] < 0x80;
        for (int k = 0; k < sl; ++k) ascii &= suf[k] < 0x80;
        for (int64_t k = 0; k < al; ++k) ascii &= ab[k] < 0x80;
        if (!ascii) {
          unsure = true;
        } else {
          if (norm == 1) {  // TRIM: str.strip()
            while (lo < hi && py_space(tb[lo])) ++lo;
            while (hi > lo && py_space(tb[hi - 1])) --hi;
          }
          eq = (int64_t)pl + (hi - lo) + sl == al;
          for (int k = 0; eq && k < pl; ++k) eq = pre[k] == ab[k];
          for (int64_t k = lo; eq && k < hi; ++k) {
            uint8_t c = tb[k];
            if (norm == 2 && c >= 'A' && c <= 'Z') c += 32;  // LOWERCASE
            eq = c == ab[pl + (k - lo)];
          }
          for (int k = 0; eq && k < sl; ++k) eq = suf[k] == ab[pl + (hi - lo) + k];
        }
      }
    }
    if (D.eq) D.eq[t] = eq ? 1 : (unsure ? 2 : 0);
    if (eq) atomicAdd(reinterpret_cast<unsigned long long*>(D.hits + h), 1ull);
    if (unsure) atomicAdd(reinterpret_cast<unsigned long long*>(D.unsure + h), 1ull);
  }
}

__global__ void key_lookup_kernel(const paste_key_lookup_desc D) {
  unsigned long long scal = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const paste_event_ref ref = D.refs[D.tape[i]];
    const int64_t c = step_child(D.nodes, ref.node_base, 0, 0, D.key);  // -1: no dict / key
    D.out_node[i] = (int32_t)c;
    if (c >= 0 && load_node(D.nodes, ref.node_base + c).type() < PASTE_T_LIST) ++scal;
  }
  for (int o = 16; o; o >>= 1) scal += __shfl_down_sync(0xffffffffu, scal, o);
  if ((threadIdx.x & 31) == 0 && scal) atomicAdd(reinterpret_cast<unsigned long long*>(D.n_scalar), scal);
}

}  // namespace paste

using namespace paste;

extern "C" int paste_tape_key_lookup(const paste_key_lookup_desc* d, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null descriptor");
  if (d->n == 0) return PASTE_OK;
  PASTE_REQUIRE(d->nodes && d->refs && d->tape && d->out_node && d->n_scalar, "null array");
  int64_t blocks = (d->n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  key_lookup_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(*d);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

extern "C" int paste_holds(const paste_holds_desc* d, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null descriptor");
  const int64_t total = d->n_hyp * d->n_occ;
  if (total == 0) return PASTE_OK;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  holds_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(*d);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
