// K5 leaf_scan and the resolve kernel over payload tapes.
//
// leaf_scan -- candidate_paths (mappings.py:237-266): the pre-order DFS that
// visits at most node_budget nodes and collects the scalar leaves equal to a
// target (values_equal, events.py:125-130).  On the tape the DFS order IS the
// node order, so a warp sweeps the first min(n_nodes, budget) nodes of one
// payload, 32 at a time, and compacts the matches in order with a ballot;
// truncated = n_nodes > budget.  Equality on canonical scalar bytes: same
// type class (str / int / float / bool value / null), same canonical bytes
// (NFC for strings), never NaN.
//
// resolve -- evaluate()'s expression resolution (mappings.py:143-194) for
// explicit (binding, source event, history) queries: the fallback index
// counts FAIL events of fail_tool after the source in its history.
#include "common.cuh"

namespace paste {

__device__ __forceinline__ int type_class(int t) {
  // TRUE and FALSE are distinct values of one class; compare them by type id
  return t;
}

__device__ __forceinline__ const uint8_t* canon_bytes(const uint8_t* bytes, int64_t byte_base,
                                                      const Node& nd, uint32_t* len) {
  const uint8_t* p = bytes + byte_base + nd.a;
  if (nd.type() == PASTE_T_STR && (nd.flags() & PASTE_F_NFC)) {
    const uint8_t* q = p + nd.b;  // [raw][u32 nfc_len][nfc]
    *len = (uint32_t)q[0] | ((uint32_t)q[1] << 8) | ((uint32_t)q[2] << 16) | ((uint32_t)q[3] << 24);
    return q + 4;
  }
  *len = nd.b;
  return p;
}

// A candidate is a leaf of the target's type class with the target's
// canonical length; only candidates need a byte comparison.  They are rare
// per 32-node sweep (a url_list has a third of its nodes as same-length
// strings), so each warp queues candidate node indices in shared memory (in
// node order) and compares 32 at a time, one per lane: full lanes instead of
// a few active lanes per sweep.  Matches are emitted in queue order = node
// order = pre-order.
constexpr int LS_T = 256;
constexpr int LS_TW = 64;  // target words staged per warp (targets up to 256 bytes)

// candidate bytes == the staged (zero-padded) target words, 8 bytes per check
__device__ __forceinline__ bool eq_target(const uint8_t* a, const uint32_t* tw, int len) {
  // 8 bytes a step; the staged target words are zero past its end
  for (int k = 0; k < len; k += 8) {
    const int r = len - k < 8 ? len - k : 8;
    const uint64_t t = (uint64_t)tw[k >> 2] | ((uint64_t)tw[(k >> 2) + 1] << 32);
    if (ld_part8(a + k, r) != t) return false;
  }
  return true;
}

__global__ void __launch_bounds__(LS_T) leaf_scan_kernel(const paste_leaf_scan_desc D) {
  __shared__ int32_t queue[LS_T / 32][64];
  __shared__ uint32_t tword[LS_T / 32][LS_TW];
  const int64_t q = (int64_t)blockIdx.x * (LS_T / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  int32_t* wq = queue[threadIdx.x / 32];
  uint32_t* tw = tword[threadIdx.x / 32];
  if (q >= D.n_queries) return;
  const paste_event_ref ref = D.refs[D.event[q]];
  const Node root = load_node(D.nodes, ref.node_base);
  const int64_t n_nodes = root.size();
  const int limit = (int)(n_nodes < D.node_budget ? n_nodes : D.node_budget);
  // target scalar
  const int tt = D.target_type[q];
  const uint8_t* tb = D.target_bytes + D.target_off[q];
  const uint32_t tl = (uint32_t)(D.target_off[q + 1] - D.target_off[q]);
  const bool tnan = D.target_nan[q] != 0;
  const bool no_bytes = tt == PASTE_T_NULL || tt == PASTE_T_TRUE || tt == PASTE_T_FALSE;
  const bool staged = tl <= 4 * LS_TW;
  if (staged)
    for (int j = lane; j < LS_TW; j += 32) {
      const int r = (int)tl - 4 * j;
      tw[j] = r > 0 ? ld_part(tb + 4 * j, r < 4 ? r : 4) : 0u;
    }
  __syncwarp();
  int64_t n_out = 0;
  const int64_t out0 = D.out_off[q], cap = D.out_off[q + 1] - out0;
  const paste_tape_node* nodes = D.nodes + ref.node_base;
  const uint8_t* bytes = D.bytes + ref.byte_base;
  if (tnan || tt < 0 || tt >= PASTE_T_LIST) goto done;
  {
    int qn = 0;  // queued candidates (warp-uniform)
    for (int base = 0; base < limit; base += 32) {
      const int i = base + lane;
      bool cand = false;
      if (i < limit) {
        const Node nd = load_node(nodes, i);
        const int t = nd.type();
        if (type_class(t) == tt && !(nd.flags() & PASTE_F_NAN)) {
          if (no_bytes) {
            cand = true;
          } else {
            uint32_t len;
            canon_bytes(bytes, 0, nd, &len);
            cand = len == tl;
          }
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, cand);
      if (cand) wq[qn + __popc(m & ((1u << lane) - 1))] = i;
      qn += __popc(m);
      const bool last = base + 32 >= limit;
      while (qn >= 32 || (last && qn > 0)) {
        __syncwarp();
        const int k = qn < 32 ? qn : 32;
        bool eq = false;
        int32_t idx = 0;
        if (lane < k) {
          idx = wq[lane];
          if (no_bytes) {
            eq = true;
          } else {
            const Node nd = load_node(nodes, idx);
            uint32_t len;
            const uint8_t* bp = canon_bytes(bytes, 0, nd, &len);
            eq = staged ? eq_target(bp, tw, (int)len) : bytes_eq(bp, tb, len);
          }
        }
        const unsigned em = __ballot_sync(0xffffffffu, eq);
        if (eq) {
          const int64_t slot = n_out + __popc(em & ((1u << lane) - 1));
          if (slot < cap) D.out_nodes[out0 + slot] = idx;
        }
        n_out += __popc(em);
        __syncwarp();
        if (lane + 32 < qn) wq[lane] = wq[lane + 32];
        qn -= k;
        __syncwarp();
      }
    }
  }
done:
  if (lane == 0) {
    D.n_out[q] = n_out;
    D.truncated[q] = n_nodes > D.node_budget;
  }
}

__global__ void resolve_kernel(const paste_resolve_desc D) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= D.n_queries) return;
  const paste_binding bd = D.bindings[q];
  const int64_t nb = D.refs[D.src_event[q]].node_base;
  const int32_t* steps = D.steps;
  int64_t cur = 0;
  for (int s = 0; s < bd.step_cnt && cur >= 0; ++s)
    cur = step_child(D.nodes, nb, cur, steps[2 * (bd.step_off + s)], steps[2 * (bd.step_off + s) + 1]);
  if (bd.kind == PASTE_X_FALLBACK) {
    int fails = 0;
    const int32_t sp = D.src_pos[q];
    if (sp >= 0)
      for (int32_t h = D.hist_off[q] + sp + 1; h < D.hist_off[q + 1]; ++h) {
        const int32_t t = D.hist_tok[h];  // -1: the source event itself (skipped)
        fails += t >= 0 && (t >> 1) == bd.fail_tool && (t & 1) == 0;
      }
    if (cur >= 0) cur = bd.start_index < 0 ? -1 : step_child(D.nodes, nb, cur, 1, bd.start_index + fails);
    for (int s = 0; s < bd.suf_cnt && cur >= 0; ++s)
      cur = step_child(D.nodes, nb, cur, steps[2 * (bd.suf_off + s)], steps[2 * (bd.suf_off + s) + 1]);
  } else if (bd.kind == PASTE_X_FORMAT && cur >= 0) {
    const int t = load_node(D.nodes, nb + cur).type();
    if (t != PASTE_T_STR && t != PASTE_T_INT && t != PASTE_T_FLOAT) cur = -1;
  }
  D.result[q] = cur;
}

// ---------------------------------------------------------------------------
// Shape-shared leaf scan.  With shape-interned tapes many payloads share one
// node array, and which of its nodes can equal a target -- same type class,
// same canonical length, not NaN, within the node budget, in pre-order --
// depends only on (node array, target type, target length).  Queries are
// grouped by that key on the host; one CTA per group scans the node array
// once and writes the group's ordered candidate list, then one warp per
// query compares only those candidates with its own payload bytes.  Strings
// whose NFC form differs keep their canonical length in the per-payload
// bytes, so they stay candidates and are length-checked per payload.
// ---------------------------------------------------------------------------
// One CTA per group: the first min(n_nodes, budget) nodes are cut into
// LS_T / 32 contiguous segments, each warp lists its segment's candidates,
// and a block scan of the segment counts places them in pre-order.
__global__ void __launch_bounds__(LS_T) leaf_candidates_kernel(const paste_leaf_scan_desc D,
                                                               const int32_t* group_rep,
                                                               int64_t n_groups, int64_t cap,
                                                               int32_t* cand, int32_t* cand_n) {
  constexpr int NW = LS_T / 32;
  __shared__ int s_cnt[NW];
  const int64_t g = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t q = group_rep[g];
  const paste_event_ref ref = D.refs[D.event[q]];
  const Node root = load_node(D.nodes, ref.node_base);
  const int64_t n_nodes = root.size();
  const int limit = (int)(n_nodes < D.node_budget ? n_nodes : D.node_budget);
  const int tt = D.target_type[q];
  const uint32_t tl = (uint32_t)(D.target_off[q + 1] - D.target_off[q]);
  const bool no_bytes = tt == PASTE_T_NULL || tt == PASTE_T_TRUE || tt == PASTE_T_FALSE;
  const bool live = !D.target_nan[q] && tt >= 0 && tt < PASTE_T_LIST;
  const paste_tape_node* nodes = D.nodes + ref.node_base;
  const int seg = (limit + NW - 1) / NW;
  const int lo = warp * seg, hi = lo + seg < limit ? lo + seg : limit;
  auto is_cand = [&](int i) {
    const Node nd = load_node(nodes, i);
    const int t = nd.type();
    return type_class(t) == tt && !(nd.flags() & PASTE_F_NAN) &&
           (no_bytes || (nd.flags() & PASTE_F_NFC) || nd.b == tl);
  };
  // pass 1: this warp's candidate count
  int cnt = 0;
  for (int base = lo; live && base < hi; base += 32)
    cnt += __popc(__ballot_sync(0xffffffffu, base + lane < hi && is_cand(base + lane)));
  if (lane == 0) s_cnt[warp] = cnt;
  __syncthreads();
  int off = 0, total = 0;
  for (int w = 0; w < NW; ++w) {
    off += w < warp ? s_cnt[w] : 0;
    total += s_cnt[w];
  }
  // pass 2: write in order (L1-hot re-read of the segment)
  int32_t* out = cand + g * cap;
  for (int base = lo; live && base < hi; base += 32) {
    const bool c = base + lane < hi && is_cand(base + lane);
    const unsigned m = __ballot_sync(0xffffffffu, c);
    const int at = off + __popc(m & ((1u << lane) - 1));
    if (c && at < cap) out[at] = base + lane;
    off += __popc(m);
  }
  if (threadIdx.x == 0) cand_n[g] = total < cap ? total : (int32_t)cap;
}

__global__ void __launch_bounds__(LS_T) leaf_match_kernel(const paste_leaf_scan_desc D,
                                                          const int32_t* group, int64_t cap,
                                                          const int32_t* cand,
                                                          const int32_t* cand_n) {
  __shared__ uint32_t tword[LS_T / 32][LS_TW];
  const int64_t q = (int64_t)blockIdx.x * (LS_T / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  uint32_t* tw = tword[threadIdx.x / 32];
  if (q >= D.n_queries) return;
  const paste_event_ref ref = D.refs[D.event[q]];
  const int tt = D.target_type[q];
  const uint8_t* tb = D.target_bytes + D.target_off[q];
  const uint32_t tl = (uint32_t)(D.target_off[q + 1] - D.target_off[q]);
  const bool no_bytes = tt == PASTE_T_NULL || tt == PASTE_T_TRUE || tt == PASTE_T_FALSE;
  const bool staged = tl <= 4 * LS_TW;
  if (staged)
    for (int j = lane; j < LS_TW; j += 32) {
      const int r = (int)tl - 4 * j;
      tw[j] = r > 0 ? ld_part(tb + 4 * j, r < 4 ? r : 4) : 0u;
    }
  __syncwarp();
  const int64_t g = group[q];
  const int32_t* list = cand + g * cap;
  const int nc = cand_n[g];
  const paste_tape_node* nodes = D.nodes + ref.node_base;
  const uint8_t* bytes = D.bytes + ref.byte_base;
  const int64_t out0 = D.out_off[q], ocap = D.out_off[q + 1] - out0;
  int64_t n_out = 0;
  for (int base = 0; base < nc; base += 32) {
    bool eq = false;
    int32_t idx = 0;
    if (base + lane < nc) {
      idx = __ldg(list + base + lane);
      if (no_bytes) {
        eq = true;
      } else {
        const Node nd = load_node(nodes, idx);
        uint32_t len;
        const uint8_t* bp = canon_bytes(bytes, 0, nd, &len);
        eq = len == tl && (staged ? eq_target(bp, tw, (int)len) : bytes_eq(bp, tb, len));
      }
    }
    const unsigned em = __ballot_sync(0xffffffffu, eq);
    if (eq) {
      const int64_t slot = n_out + __popc(em & ((1u << lane) - 1));
      if (slot < ocap) D.out_nodes[out0 + slot] = idx;
    }
    n_out += __popc(em);
  }
  if (lane == 0) {
    D.n_out[q] = n_out;
    D.truncated[q] = load_node(D.nodes, ref.node_base).size() > (uint64_t)D.node_budget;
  }
}

}  // namespace paste

using namespace paste;

extern "C" int64_t paste_leaf_scan_shared_bytes(int64_t n_groups, int64_t node_budget) {
  return n_groups <= 0 ? 0 : n_groups * (node_budget + 1) * (int64_t)sizeof(int32_t);
}

extern "C" int paste_leaf_scan_shared(const paste_leaf_scan_desc* d, const int32_t* group,
                                      int64_t n_groups, const int32_t* group_rep, void* scratch,
                                      void* stream) {
  using namespace paste;
  reset_launches();
  PASTE_REQUIRE(d != nullptr && group != nullptr && group_rep != nullptr && scratch != nullptr,
                "null argument");
  PASTE_REQUIRE(d->node_budget >= 0 && d->node_budget < (1ll << 30), "node budget out of range");
  if (d->n_queries == 0) return PASTE_OK;
  const int64_t cap = d->node_budget;
  int32_t* cand_n = static_cast<int32_t*>(scratch);
  int32_t* cand = cand_n + n_groups;
  const int warps = LS_T / 32;
  leaf_candidates_kernel<<<(unsigned)n_groups, LS_T, 0, (cudaStream_t)stream>>>(
      *d, group_rep, n_groups, cap > 0 ? cap : 1, cand, cand_n);
  leaf_match_kernel<<<(unsigned)((d->n_queries + warps - 1) / warps), LS_T, 0,
                      (cudaStream_t)stream>>>(*d, group, cap > 0 ? cap : 1, cand, cand_n);
  count_launch(2);
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

extern "C" int paste_leaf_scan(const paste_leaf_scan_desc* d, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null descriptor");
  if (d->n_queries == 0) return PASTE_OK;
  const int warps = 8;
  const int64_t blocks = (d->n_queries + warps - 1) / warps;
  leaf_scan_kernel<<<(unsigned)blocks, warps * 32, 0, (cudaStream_t)stream>>>(*d);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

extern "C" int paste_resolve(const paste_resolve_desc* d, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null descriptor");
  if (d->n_queries == 0) return PASTE_OK;
  const int threads = 128;
  resolve_kernel<<<(unsigned)((d->n_queries + threads - 1) / threads), threads, 0,
                   (cudaStream_t)stream>>>(*d);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
