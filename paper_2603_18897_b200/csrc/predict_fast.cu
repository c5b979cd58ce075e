// K4 fast path: match-table predict + streamed admit, no local memory.
//
// Same results as predict_kernel (predict.cu; reference prediction.py:76-118,
// mining.py:119-156, mappings.py:143-223, policy.py:207-244), restructured for
// sm_100a:
//
// * Pool compilation (build_match_table_kernel): which patterns match at an
//   anchor, their rank order and the matched position of every binding's
//   source depend only on the newest G tool tokens (match_at never looks
//   further back than k events, mining.py:142; the suffix relation needs the
//   newest max_ctx).  One thread per key runs the bucket scan once and
//   stores the first K matches -- with the pattern fields the live kernel
//   needs and the age of every binding's source -- so the live kernel does
//   one L2-resident table read per session instead of a divergent bucket
//   scan followed by dependent pattern loads.
// * Window rings may be slot-major ([W][n]): sessions that step together
//   (a batch of tool completions) read and write contiguous 128-byte lines.
//   Each thread gathers its newest G tool events (token, ring slot) into a
//   G-deep shared-memory row, so no array ever lands in local memory.
// * Admit is streamed in rank order.  Candidates arrive sorted by p
//   descending, so for a tool whose benefit b is >= 0 (or NaN) the utility
//   p*b is non-increasing and the reference's strict (utility, p,
//   -created_at) arbitration (_beats, policy.py:239-244) keeps the FIRST
//   allowed candidate of the tool: a seen-tool bitmask replaces the K x K
//   comparison.  Tools with a negative benefit (or ids >= 64) take the exact
//   comparison path against the incumbent's record.
#include "common.cuh"
#include "fast.cuh"

namespace paste {

constexpr int FT = 128;         // threads per CTA
constexpr int MT_MAX_BIND = 8;  // 4-bit source ages per binding in a uint32

struct FastParams {
  paste_pool_desc pool;
  paste_windows win;
  paste_admit_desc adm;
  paste_predict_out out;
  int G;    // gathered tool events: min(k | max_ctx, W)
  int row;  // smem words per thread (2G + 1)
};

// ---------------------------------------------------------------------------
// match-table build: one thread per key (the reference's bucket scan, run
// once per distinct token context)
// ---------------------------------------------------------------------------
__global__ void build_match_table_kernel(const paste_pool_desc pool, int K, int G,
                                         int64_t n_keys, uint8_t* table) {
  const int64_t key = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (key >= n_keys) return;
  const int S = pool.n_bucket_sigs, base = S + 1;
  int32_t tok[16];  // by age; -2 = no event / unknown signature
  {  // key = anchor + S * sum_{a>=1} code(a) * (S+1)^(a-1)
    tok[0] = (int)(key % S);
    int64_t k = key / S;
    for (int a = 1; a < G; ++a) {
      const int c = (int)(k % base);
      k /= base;
      tok[a] = c == S ? -2 : c;
    }
  }
  int32_t* hdr = reinterpret_cast<int32_t*>(table + key * mt_stride(K));
  MTRecord* rec = reinterpret_cast<MTRecord*>(hdr + 4);
  int n_match = 0, n_err = 0;
  const int a = tok[0];
  const int m = G;  // absent positions behave as never-matching tokens
#define TK(p) tok[m - 1 - (p)]
  const bool anchored = pool.relation == PASTE_REL_ANCHORED;
  for (int bi = pool.bucket_off[a]; bi < pool.bucket_off[a + 1]; ++bi) {
    const int pid = pool.bucket_pat[bi];
    const paste_pattern pt = pool.patterns[pid];
    const int n = pt.ctx_len;
    const int32_t* ctx = pool.ctx_sig + pt.ctx_off;
    int pos_of[16];
    bool ok;
    if (anchored) {
      if (n > 16) continue;
      pos_of[n - 1] = m - 1;
      int j = n - 2, pos = m - 2;
      while (j >= 0 && pos >= 0) {
        if (TK(pos) == ctx[j]) pos_of[j--] = pos;
        --pos;
      }
      ok = j < 0;
    } else {
      ok = n <= m;
      for (int i = 0; ok && i < n - 1; ++i) ok = TK(m - n + i) == ctx[i];
      if (ok)
        for (int i = 0; i < n; ++i) pos_of[i] = m - n + i;
    }
    if (!ok) continue;
    if (pt.flags & PASTE_PF_STRUCT_ERR) {
      ++n_err;
      continue;
    }
    if (n_match < K) {
      uint32_t src = 0;
      for (int b = 0; b < pt.n_bind && b < MT_MAX_BIND; ++b) {
        const int cp = pool.bindings[pt.bind_off + b].ctx_pos;
        src |= (uint32_t)(m - 1 - pos_of[cp]) << (4 * b);  // age of the source
      }
      MTRecord r;
      r.pid = pid;
      r.src = src;
      r.tool = pt.target_tool;
      r.nb_flags = pt.n_bind | (pt.flags << 16);
      r.bind_off = pt.bind_off;
      r.pad = 0;
      r.p = pt.p;
      rec[n_match] = r;
    }
    ++n_match;
  }
#undef TK
  hdr[0] = n_match;
  hdr[1] = n_err;
  hdr[2] = 0;
  hdr[3] = 0;
}

static int64_t keys_for(const paste_pool_desc* pool, int G) {
  const int64_t base = (int64_t)pool->n_bucket_sigs + 1;
  int64_t n = pool->n_bucket_sigs;
  for (int a = 1; a < G; ++a) {
    n *= base;
    if (n > ((int64_t)1 << 40)) return -1;
  }
  return n;
}

static int gather_depth(const paste_pool_desc* pool, int W) {
  const int g = pool->relation == PASTE_REL_ANCHORED ? pool->k : pool->max_ctx;
  return g < W ? g : W;
}

}  // namespace paste

extern "C" int64_t paste_match_table_bytes(const paste_pool_desc* pool, int32_t max_candidates,
                                           int32_t window_capacity) {
  using namespace paste;
  if (!pool || max_candidates < 1 || window_capacity < 1 || window_capacity > 16) return -1;
  if (pool->max_bindings > MT_MAX_BIND || pool->n_bucket_sigs < 1) return -1;
  const int G = gather_depth(pool, window_capacity);
  if (G < 1 || G > 16) return -1;
  const int64_t keys = keys_for(pool, G);
  if (keys < 0) return -1;
  const int64_t bytes = keys * mt_stride(max_candidates);
  if (bytes > ((int64_t)1 << 30)) return -1;  // keep tables L2/HBM friendly
  return bytes;
}

extern "C" int paste_build_match_table(const paste_pool_desc* pool, int32_t max_candidates,
                                       int32_t window_capacity, void* table, void* stream) {
  using namespace paste;
  reset_launches();
  const int64_t bytes = paste_match_table_bytes(pool, max_candidates, window_capacity);
  if (bytes < 0) {
    set_error("pool is outside the match-table envelope");
    return PASTE_ERR_UNSUPPORTED;
  }
  PASTE_REQUIRE(table != nullptr, "null table");
  const int G = gather_depth(pool, window_capacity);
  const int64_t keys = keys_for(pool, G);
  const int threads = 128;
  build_match_table_kernel<<<(unsigned)((keys + threads - 1) / threads), threads, 0,
                             (cudaStream_t)stream>>>(*pool, max_candidates, G, keys,
                                                     static_cast<uint8_t*>(table));
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

namespace paste {

struct OutIdx {  // record addressing for one session (session- or slot-major)
  int64_t obase, ostride, abase;
  int B;
  __device__ __forceinline__ int64_t o(int i) const { return obase + (int64_t)i * ostride; }
  __device__ __forceinline__ int64_t a(int i, int b) const {
    return abase + (int64_t)(i * B + b) * ostride;
  }
};

// Streamed admit of candidate `i` (policy.py:207-236).
__device__ __forceinline__ void admit_one(const FastParams& P, const OutIdx& X, int i, int tool,
                                          int comp, double p, int& n_act, uint64_t& seen) {
  if (tool >= P.adm.n_tools || !__ldg(P.adm.allow + tool)) return;
  const int implied = comp == PASTE_C_FULL ? 3 : 1;
  const int cap = __ldg(P.adm.max_level + tool);
  const int level = cap < implied ? cap : implied;
  const double bene = __ldg(P.adm.benefit + tool);
  const double util = __dmul_rn(p, bene);
  if (!(bene < 0.0) && tool < 64) {
    if ((seen >> tool) & 1ull) return;  // an earlier (higher-p) candidate wins
    seen |= 1ull << tool;
    const int64_t o = X.o(n_act);
    P.out.act_pred[o] = (int16_t)i;
    P.out.act_level[o] = (uint8_t)level;
    P.out.act_util[o] = util;
    ++n_act;
    return;
  }
  int j = 0;  // exact arbitration against the incumbent (rare)
  for (; j < n_act; ++j) {
    const int ip = P.out.act_pred[X.o(j)];
    if (P.pool.patterns[P.out.pred_pat[X.o(ip)]].target_tool == tool) break;
  }
  const int64_t o = X.o(j);
  if (j == n_act) {
    P.out.act_pred[o] = (int16_t)i;
    P.out.act_level[o] = (uint8_t)level;
    P.out.act_util[o] = util;
    ++n_act;
    return;
  }
  const double iu = P.out.act_util[o];
  const double ipp = P.pool.patterns[P.out.pred_pat[X.o(P.out.act_pred[o])]].p;
  if ((util != iu) ? (util > iu) : (p > ipp)) {
    P.out.act_pred[o] = (int16_t)i;
    P.out.act_level[o] = (uint8_t)level;
    P.out.act_util[o] = util;
  }
}

// observe (PredictionWindow.observe) + gather the newest G tool events of
// session `sess` into its shared-memory row (gt: tokens by age, age 0 =
// newest; gs: their ring slots).  Returns how many were gathered.
__device__ __forceinline__ int observe_gather(const FastParams& P, int64_t sess, int32_t* gt,
                                              int64_t& rbase, int64_t& rstride) {
  const int64_t n = P.win.n_sessions;
  const int W = P.win.capacity, G = P.G;
  int32_t* gs = gt + G;  // ring slots of the gathered tokens
  rbase = P.win.stream_end ? P.win.stream_end[sess] - P.win.count[sess]
                           : (P.win.slot_major ? sess : sess * W);
  rstride = (P.win.slot_major && !P.win.stream_end) ? n : 1;
  int64_t cnt = P.win.count[sess];
  int head = (int)(cnt % W);  // next slot to write
  int32_t new_t = -1;
  if (P.win.new_tok != nullptr) {  // observe (PredictionWindow.observe)
    const int64_t ev = P.win.new_evt_base + sess;
    paste_event_ref r;
    if (P.win.new_node != nullptr) {
      r.node_base = P.win.new_node[sess];
      r.byte_base = 0;
    } else {
      r = P.win.new_ref[sess];
    }
    r.byte_base += P.win.new_byte_base;
    P.win.refs[ev] = r;
    new_t = P.win.new_tok[sess];
    const int64_t at = rbase + head * rstride;
    P.win.tok[at] = new_t;
    P.win.evt[at] = (int32_t)ev;
    ++cnt;
    P.win.count[sess] = cnt;
    head = head + 1 == W ? 0 : head + 1;
  }
  const int len = (int)(cnt < W ? cnt : W);
  int m = 0;
  int slot = head;
  for (int i = 0; i < len && m < G; ++i) {
    slot = slot == 0 ? W - 1 : slot - 1;
    const int32_t t = (i == 0 && P.win.new_tok != nullptr) ? new_t : P.win.tok[rbase + slot * rstride];
    if (t >= 0) {
      gt[m] = t;
      gs[m] = slot;
      ++m;
    }
  }
  return m;
}

// match-table key / entry of the gathered tokens (the newest G tool tokens)
__device__ __forceinline__ int64_t table_key(const FastParams& P, const int32_t* gt, int m) {
  const int S = P.pool.n_bucket_sigs, G = P.G;
  int64_t key = gt[0], mult = S;
  for (int a = 1; a < G; ++a) {
    const int t = a < m ? gt[a] : S;
    key += (int64_t)(t < S ? t : S) * mult;
    mult *= (S + 1);
  }
  return key;
}

__device__ __forceinline__ const uint8_t* table_entry(const FastParams& P, const int32_t* gt,
                                                      int m) {
  const int S = P.pool.n_bucket_sigs, G = P.G;
  int64_t key = gt[0], mult = S;
  for (int a = 1; a < G; ++a) {
    const int t = a < m ? gt[a] : S;
    key += (int64_t)(t < S ? t : S) * mult;
    mult *= (S + 1);
  }
  return static_cast<const uint8_t*>(P.pool.match_table) + key * mt_stride(P.pool.mt_k);
}

template <bool TABLE>
__device__ __forceinline__ void predict_session(const FastParams& P, int64_t sess, int32_t* gt,
                                                uint64_t* memo) {
  const int64_t n = P.win.n_sessions;
  const int G = P.G;
  int32_t* gs = gt + G;  // ring slots of the gathered tokens
  const int K = P.out.max_candidates;
  OutIdx X;
  X.B = P.out.max_bindings;
  X.ostride = P.out.slot_major ? n : 1;
  X.obase = P.out.slot_major ? sess : sess * K;
  X.abase = P.out.slot_major ? sess : sess * K * X.B;
  int64_t rbase, rstride;
  const int m = observe_gather(P, sess, gt, rbase, rstride);

  const paste_pool_desc& pool = P.pool;
  const bool admit = P.adm.enabled != 0;
  int n_pred = 0, n_err = 0, n_act = 0;
  uint64_t seen = 0;  // tools (< 64) that already hold an action
  const int S = pool.n_bucket_sigs;

  if (m > 0 && gt[0] < S) {
    if (TABLE) {
      // ---- table path: one entry per distinct token context ---------------
      const uint8_t* e = table_entry(P, gt, m);
      const int2 hdr = __ldg(reinterpret_cast<const int2*>(e));
      const MTRecord* recs = reinterpret_cast<const MTRecord*>(e + 16);
      n_err = hdr.y;
      const int nm = hdr.x < K ? hdr.x : K;
      for (int i = 0; i < nm; ++i) {
        const int4 r0 = __ldg(reinterpret_cast<const int4*>(recs + i));
        const int4 r1 = __ldg(reinterpret_cast<const int4*>(recs + i) + 1);
        const int pid = r0.x, tool = r0.z, n_bind = r0.w & 0xffff, pflags = r0.w >> 16;
        const uint32_t src = (uint32_t)r0.y;
        const int bind_off = r1.x;
        const double p = __hiloint2double(r1.w, r1.z);
        int comp = PASTE_C_TOOL_ONLY;
        if (pflags & PASTE_PF_HAS_MAPPING) {
          comp = PASTE_C_FULL;
          for (int b = 0; b < n_bind; ++b) {
            const paste_binding bd = pool.bindings[bind_off + b];
            const int age = (src >> (4 * b)) & 15;
            const int32_t ev = P.win.evt[rbase + gs[age] * rstride];
            const int64_t r = resolve_fast(P.win, pool.steps, bd, bind_off + b, ev, age, gt, memo);
            if (r < 0) comp = PASTE_C_PARTIAL;
            P.out.pred_arg[X.a(i, b)] = r;
          }
        }
        const int64_t o = X.o(i);
        P.out.pred_pat[o] = pid;
        P.out.pred_comp[o] = (uint8_t)comp;
        if (admit) admit_one(P, X, i, tool, comp, p, n_act, seen);
      }
      n_pred = nm;
    } else {
      // ---- scan path (no table): bucket in rank order ------------------------
      const int a = gt[0];
      const int b0 = __ldg(pool.bucket_off + a), b1 = __ldg(pool.bucket_off + a + 1);
      const bool scan_all = __ldg(pool.bucket_scan_all + a) != 0;
      const bool anchored = pool.relation == PASTE_REL_ANCHORED;
#define GT(p) gt[m - 1 - (p)]
      for (int bi = b0; bi < b1; ++bi) {
        const int pid = __ldg(pool.bucket_pat + bi);
        const int4 h = __ldg(reinterpret_cast<const int4*>(pool.patterns + pid));
        const int nctx = h.y, tool = h.z, bind_off = h.w;
        const int32_t* ctx = pool.ctx_sig + h.x;
        bool ok;
        if (anchored) {
          int j = nctx - 2, pos = m - 2;
          while (j >= 0 && pos >= 0) {
            j -= GT(pos) == __ldg(ctx + j);
            --pos;
          }
          ok = j < 0;
        } else {
          ok = nctx <= m;
          for (int i = 0; ok && i < nctx - 1; ++i) ok = GT(m - nctx + i) == __ldg(ctx + i);
        }
        if (!ok) continue;
        const int4 h2 = __ldg(reinterpret_cast<const int4*>(pool.patterns + pid) + 1);
        const int n_bind = h2.x, pflags = h2.y;
        const double p = __hiloint2double(h2.w, h2.z);
        if (pflags & PASTE_PF_STRUCT_ERR) {
          ++n_err;
          continue;
        }
        if (n_pred >= K) {
          if (!scan_all) break;
          continue;
        }
        int comp = PASTE_C_TOOL_ONLY;
        if (pflags & PASTE_PF_HAS_MAPPING) {
          comp = PASTE_C_FULL;
          for (int b = 0; b < n_bind; ++b) {
            const paste_binding bd = pool.bindings[bind_off + b];
            int src;  // matched position of context element ctx_pos
            if (!anchored) {
              src = m - nctx + bd.ctx_pos;
            } else if (bd.ctx_pos == nctx - 1) {
              src = m - 1;
            } else {
              int j = nctx - 2, pos = m - 2;
              src = 0;
              while (j >= 0 && pos >= 0) {
                if (GT(pos) == __ldg(ctx + j)) {
                  if (j == bd.ctx_pos) { src = pos; break; }
                  --j;
                }
                --pos;
              }
            }
            const int age = m - 1 - src;
            const int32_t ev = P.win.evt[rbase + gs[age] * rstride];
            const int64_t r = resolve_fast(P.win, pool.steps, bd, bind_off + b, ev, age, gt, memo);
            if (r < 0) comp = PASTE_C_PARTIAL;
            P.out.pred_arg[X.a(n_pred, b)] = r;
          }
        }
        const int64_t o = X.o(n_pred);
        P.out.pred_pat[o] = pid;
        P.out.pred_comp[o] = (uint8_t)comp;
        if (admit) admit_one(P, X, n_pred, tool, comp, p, n_act, seen);
        ++n_pred;
        if (n_pred >= K && !scan_all) break;
      }
#undef GT
    }
  }
  P.out.n_pred[sess] = n_pred;
  P.out.struct_err[sess] = n_err;
  if (admit) P.out.n_act[sess] = n_act;
}


// ---------------------------------------------------------------------------
// Warp-cooperative table path.  Lane-per-session resolution leaves most
// lanes idle (about 7 of 32 sessions have a mapped candidate at a given rank)
// so the argument walks -- the bulk of the instructions -- run from a
// per-warp queue instead, one binding per lane:
//   A. lane per session: observe, gather, table entry; per candidate rank the
//      pattern id is written and the mapped bindings are queued (event,
//      binding, owner lane / rank / slot / source age);
//   B. whole warp: full rounds of 32 queued bindings are resolved (walk memo
//      as before) and written; an unresolved one marks its candidate PARTIAL
//      in the owner's shared-memory mask;
//   C. lane per session: completeness codes and the streamed admit.
// ---------------------------------------------------------------------------
constexpr int RQ = 32 + 32 * MT_MAX_BIND;  // queue entries per warp
constexpr int COOP_MAX_K = 64;             // candidate rank fits 6 bits

struct ResolveQueue {
  uint32_t bind[RQ];
  uint32_t meta[RQ];   // owner lane | rank << 5 | slot << 11 | source age << 14
  int64_t rbase[32];   // ring addressing of every lane's session
  int64_t rstride[32];
  unsigned long long part[32];  // ranks with an unresolved binding, per lane
};

__host__ __device__ inline size_t coop_smem_bytes(int row) {
  return sizeof(uint64_t) * MEMO + sizeof(int32_t) * FT * row +
         sizeof(ResolveQueue) * (FT / 32);
}

__device__ __forceinline__ OutIdx out_idx(const FastParams& P, int64_t sess) {
  const int64_t n = P.win.n_sessions;
  const int K = P.out.max_candidates;
  OutIdx X;
  X.B = P.out.max_bindings;
  X.ostride = P.out.slot_major ? n : 1;
  X.obase = P.out.slot_major ? sess : sess * K;
  X.abase = P.out.slot_major ? sess : sess * K * X.B;
  return X;
}

__device__ __forceinline__ void predict_coop(const FastParams& P, int64_t sess, bool live,
                                             int32_t* rows, uint64_t* memo, ResolveQueue& q) {
  const unsigned FULLM = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t warp_first = sess - lane;
  int32_t* gt = rows + lane * P.row;
  const paste_pool_desc& pool = P.pool;
  const OutIdx X = out_idx(P, sess);
  const bool admit = P.adm.enabled != 0;
  int64_t rbase = 0, rstride = 0;
  int nm = 0, n_err = 0, n_act = 0;
  uint64_t seen = 0;
  const MTRecord* recs = nullptr;
  if (live) {
    const int m = observe_gather(P, sess, gt, rbase, rstride);
    if (m > 0 && gt[0] < pool.n_bucket_sigs) {
      const uint8_t* e = table_entry(P, gt, m);
      const int2 hdr = __ldg(reinterpret_cast<const int2*>(e));
      recs = reinterpret_cast<const MTRecord*>(e + 16);
      n_err = hdr.y;
      nm = hdr.x < P.out.max_candidates ? hdr.x : P.out.max_candidates;
    }
  }
  q.rbase[lane] = rbase;
  q.rstride[lane] = rstride;
  q.part[lane] = 0ull;
  __syncwarp();
  const int max_nm = (int)__reduce_max_sync(FULLM, (unsigned)nm);
  int count = 0;
  int32_t* pp = P.out.pred_pat + X.obase;   // rank i's record slot, advanced per rank
  uint8_t* pc = P.out.pred_comp + X.obase;
  for (int i = 0; i < max_nm; ++i, pp += X.ostride, pc += X.ostride) {
    // ---- A: rank i of every session: records, provisional completeness
    // (FULL when mapped; B downgrades), admit, mapped bindings queued --------
    int nb = 0, bind_off = 0;
    uint32_t src = 0;
    if (i < nm) {
      const int4 r0 = __ldg(reinterpret_cast<const int4*>(recs + i));
      const int4 r1 = __ldg(reinterpret_cast<const int4*>(recs + i) + 1);
      const bool mapped = ((r0.w >> 16) & PASTE_PF_HAS_MAPPING) != 0;
      const int comp = mapped ? PASTE_C_FULL : PASTE_C_TOOL_ONLY;
      *pp = r0.x;
      *pc = (uint8_t)comp;
      if (admit) {
        const int tool = r0.z;
        const double p = __hiloint2double(r1.w, r1.z);
        if (tool < 64 && tool < P.adm.n_tools) {
          // streamed first-candidate rule inline (admit_one's fast path), with
          // the action slot advanced by pointer
          if (__ldg(P.adm.allow + tool) && !((seen >> tool) & 1ull)) {
            const double bene = __ldg(P.adm.benefit + tool);
            if (!(bene < 0.0)) {
              seen |= 1ull << tool;
              const int implied = comp == PASTE_C_FULL ? 3 : 1;
              const int cap = __ldg(P.adm.max_level + tool);
              const int64_t o = X.obase + (int64_t)n_act * X.ostride;
              P.out.act_pred[o] = (int16_t)i;
              P.out.act_level[o] = (uint8_t)(cap < implied ? cap : implied);
              P.out.act_util[o] = __dmul_rn(p, bene);
              ++n_act;
            } else {
              admit_one(P, X, i, tool, comp, p, n_act, seen);
            }
          }
        } else {
          admit_one(P, X, i, tool, comp, p, n_act, seen);
        }
      }
      if (mapped) {
        nb = r0.w & 0xffff;
        src = (uint32_t)r0.y;
        bind_off = r1.x;
      }
    }
    // offsets: one binding per candidate is the common case (ballot); wider
    // candidates add a scan
    int pos, total;
    const unsigned any = __ballot_sync(FULLM, nb > 0);
    if (__all_sync(FULLM, nb <= 1)) {
      pos = count + __popc(any & lt);
      total = __popc(any);
    } else {
      int incl = nb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULLM, incl, o);
        if (lane >= o) incl += t;
      }
      total = __shfl_sync(FULLM, incl, 31);
      pos = count + incl - nb;
    }
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      q.bind[pos + b] = (uint32_t)(bind_off + b);
      q.meta[pos + b] = (uint32_t)lane | ((uint32_t)i << 5) | ((uint32_t)b << 11) |
                        (((src >> (4 * b)) & 15u) << 14);
    }
    count += total;
    __syncwarp();
    // ---- B: full rounds of 32 bindings (and the rest after the last rank) --
    const bool last = i + 1 == max_nm;
    while (count >= 32 || (last && count > 0)) {
      const int take = count < 32 ? count : 32;
      if (lane < take) {
        const int t = count - take + lane;
        const uint32_t meta = q.meta[t];
        const int owner = meta & 31, ri = (meta >> 5) & 63, slot = (meta >> 11) & 7;
        const int age = (meta >> 14) & 15;
        const int bind = (int)q.bind[t];
        const int32_t* ogt = rows + owner * P.row;
        const int32_t ev = P.win.evt[q.rbase[owner] + ogt[P.G + age] * q.rstride[owner]];
        const paste_binding bd = pool.bindings[bind];
        const int64_t r = resolve_fast(P.win, pool.steps, bd, bind, ev, age, ogt, memo);
        const OutIdx Y = out_idx(P, warp_first + owner);
        P.out.pred_arg[Y.a(ri, slot)] = r;
        if (r < 0) {
          P.out.pred_comp[Y.o(ri)] = (uint8_t)PASTE_C_PARTIAL;
          atomicOr(q.part + owner, 1ull << ri);
        }
      }
      count -= take;
      __syncwarp();
    }
  }
  __syncwarp();
  if (!live) return;
  // ---- C: admitted PARTIAL candidates get level min(cap, WARM_ONLY) ---------
  const unsigned long long pm = q.part[lane];
  if (admit && pm) {
    for (int j = 0; j < n_act; ++j) {
      const int64_t o = X.o(j);
      const int ip = P.out.act_pred[o];
      if ((pm >> ip) & 1ull) {
        const int cap = __ldg(P.adm.max_level + __ldg(&recs[ip].tool));
        P.out.act_level[o] = (uint8_t)(cap < 1 ? cap : 1);
      }
    }
  }
  P.out.n_pred[sess] = nm;
  P.out.struct_err[sess] = n_err;
  if (admit) P.out.n_act[sess] = n_act;
}

// Persistent CTAs (grid = SMs x resident CTAs): each loops over 128-session
// chunks so its shared-memory walk memo stays warm across chunks.
template <bool TABLE>
__global__ void __launch_bounds__(FT, 8) predict_fast_kernel(const FastParams P) {
  extern __shared__ uint64_t s_mem[];
  uint64_t* memo = s_mem;
  for (int i = threadIdx.x; i < MEMO; i += FT) memo[i] = 0;
  __syncthreads();
  int32_t* rows = reinterpret_cast<int32_t*>(s_mem + MEMO);
  int32_t* gt = rows + threadIdx.x * P.row;
  const int64_t n = P.win.n_sessions;
  if (TABLE && P.out.max_candidates <= COOP_MAX_K) {
    const int warp = threadIdx.x >> 5;
    ResolveQueue* qs = reinterpret_cast<ResolveQueue*>(rows + FT * P.row);
    for (int64_t first = (int64_t)blockIdx.x * FT; first < n; first += (int64_t)gridDim.x * FT) {
      const int64_t sess = first + threadIdx.x;
      predict_coop(P, sess, sess < n, rows + warp * 32 * P.row, memo, qs[warp]);
    }
    return;
  }
  for (int64_t first = (int64_t)blockIdx.x * FT; first < n; first += (int64_t)gridDim.x * FT) {
    const int64_t sess = first + threadIdx.x;
    if (sess < n) predict_session<TABLE>(P, sess, gt, memo);
  }
}

// ---------------------------------------------------------------------------
// Fused predict + compaction (the serving path, paste_predict_compact): the
// step's records go straight into the narrow CSR streams of
// paste_compact_desc (compact.cu describes the format) instead of K fixed
// slots per session that a second kernel then compacts.  Tiles of FT
// sessions are claimed through a ticket (so every predecessor is running or
// done) and each tile runs in two phases around a decoupled look-back:
//   1. the whole step (observe, gather, match, resolve, admit), its records
//      staged per thread in shared memory, and its counts;
//   2. a block scan plus a decoupled look-back give the stream offsets and
//      the staged records are written out in the chosen widths.
// ---------------------------------------------------------------------------
struct CompactParams {
  FastParams F;
  paste_compact_desc C;
  uint64_t* ticket;
  uint64_t* tile_state;  // [tiles][LB_STRIDE]
  int64_t n_tiles;
};

__device__ __forceinline__ bool allowed_tool(const paste_admit_desc& adm, int tool) {
  return adm.enabled && tool < adm.n_tools && __ldg(adm.allow + tool);
}

// Per-thread staging of one session's records in shared memory (codes in
// the wide forms; widths are applied when the tile is flushed).
struct Stage {
  uint16_t* pred;  // [K] pattern | completeness << 14
  uint32_t* arg;   // [K * B] region << 27 | node, all-ones = unresolved / not representable
  uint8_t* act;    // [K] slot | level << 5
};

__host__ __device__ inline int stage_stride(int K, int B) {  // bytes per thread, 16-B aligned
  return (((2 * K + 3) & ~3) + 4 * K * B + ((K + 3) & ~3) + 15) & ~15;
}

// Observe, gather, match, resolve, admit and stage session `sess` (all
// lanes of the warp call this together; `live` = the lane has a session).
// Same warp-cooperative scheme as predict_coop: lane per session for the
// records and the admit, one queued binding per lane for the argument walks;
// an unresolved binding marks its candidate in the owner's PARTIAL mask and
// the owner fixes the staged completeness / action levels at the end.
// c = {predictions, arguments, actions, structural errors}.
__device__ __forceinline__ void compact_stage(const FastParams& P, int64_t sess, bool live,
                                              int32_t* rows, uint8_t* stage0, int sstride,
                                              const Stage& S, int c[4], uint64_t* memo,
                                              ResolveQueue& q, unsigned long long& wide,
                                              uint32_t& key) {
  const unsigned FULLM = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t warp_first = sess - lane;
  const int64_t n = P.win.n_sessions;
  const int K = P.out.max_candidates;
  const paste_pool_desc& pool = P.pool;
  int32_t* gt = rows + lane * P.row;
  c[0] = c[1] = c[2] = c[3] = 0;
  key = 0xffffu;
  int64_t rbase = 0, rstride = 0;
  int nm = 0;
  const MTRecord* recs = nullptr;
  if (live) {
    const int m = observe_gather(P, sess, gt, rbase, rstride);
    if (m > 0 && gt[0] < pool.n_bucket_sigs) {
      const int64_t tk = table_key(P, gt, m);
      key = (uint32_t)tk;
      const uint8_t* e = static_cast<const uint8_t*>(pool.match_table) + tk * mt_stride(pool.mt_k);
      const int2 hdr = __ldg(reinterpret_cast<const int2*>(e));
      recs = reinterpret_cast<const MTRecord*>(e + 16);
      nm = hdr.x < K ? hdr.x : K;
      c[3] = hdr.y;
    }
  }
  q.rbase[lane] = rbase;
  q.rstride[lane] = rstride;
  q.part[lane] = 0ull;
  __syncwarp();
  const int max_nm = (int)__reduce_max_sync(FULLM, (unsigned)nm);
  int na = 0, n_act = 0, count = 0;
  uint64_t seen = 0;
  const int arg_off = (2 * K + 3) & ~3;  // Stage.arg within a thread's staging
  for (int i = 0; i < max_nm; ++i) {
    int nb = 0, bind_off = 0;
    uint32_t src = 0;
    if (i < nm) {
      const int4 r0 = __ldg(reinterpret_cast<const int4*>(recs + i));
      const int4 r1 = __ldg(reinterpret_cast<const int4*>(recs + i) + 1);
      const int pid = r0.x, tool = r0.z, pflags = r0.w >> 16;
      const double p = __hiloint2double(r1.w, r1.z);
      const bool mapped = (pflags & PASTE_PF_HAS_MAPPING) != 0;
      const int comp = mapped ? PASTE_C_FULL : PASTE_C_TOOL_ONLY;  // B may downgrade
      S.pred[i] = (uint16_t)(pid | (comp << 14));
      if (mapped) {
        nb = r0.w & 0xffff;
        src = (uint32_t)r0.y;
        bind_off = r1.x;
      }
      // admit (policy.py:207-236): the streamed first-candidate rule for
      // tools with benefit >= 0 (or NaN), exact arbitration otherwise
      if (allowed_tool(P.adm, tool)) {
        const int implied = comp == PASTE_C_FULL ? 3 : 1;
        const int cap = __ldg(P.adm.max_level + tool);
        const uint8_t rec = (uint8_t)(i | ((cap < implied ? cap : implied) << 5));
        const double bene = __ldg(P.adm.benefit + tool);
        if (!(bene < 0.0) && tool < 64) {
          if (!((seen >> tool) & 1ull)) {
            seen |= 1ull << tool;
            S.act[n_act++] = rec;
          }
        } else {
          int j = 0;
          for (; j < n_act; ++j)
            if (__ldg(&recs[S.act[j] & 31].tool) == tool) break;
          if (j == n_act) {
            S.act[n_act++] = rec;
          } else {
            const int ip = S.act[j] & 31;
            const double ipp = __ldg(&recs[ip].p);
            const double util = __dmul_rn(p, bene), iu = __dmul_rn(ipp, bene);
            if ((util != iu) ? (util > iu) : (p > ipp)) S.act[j] = rec;
          }
        }
      }
    }
    int pos, total;
    const unsigned any = __ballot_sync(FULLM, nb > 0);
    if (__all_sync(FULLM, nb <= 1)) {
      pos = count + __popc(any & lt);
      total = __popc(any);
    } else {
      int incl = nb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULLM, incl, o);
        if (lane >= o) incl += t;
      }
      total = __shfl_sync(FULLM, incl, 31);
      pos = count + incl - nb;
    }
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      q.bind[pos + b] = (uint32_t)(bind_off + b);
      q.meta[pos + b] = (uint32_t)lane | ((uint32_t)i << 5) | (((src >> (4 * b)) & 15u) << 14) |
                        ((uint32_t)(na + b) << 18);
    }
    na += nb;
    count += total;
    __syncwarp();
    const bool last = i + 1 == max_nm;
    while (count >= 32 || (last && count > 0)) {
      const int take = count < 32 ? count : 32;
      if (lane < take) {
        const int t = count - take + lane;
        const uint32_t meta = q.meta[t];
        const int owner = meta & 31, ri = (meta >> 5) & 63, age = (meta >> 14) & 15;
        const int apos = (meta >> 18) & 63;
        const int bind = (int)q.bind[t];
        const int32_t* ogt = rows + owner * P.row;
        const int32_t ev = P.win.evt[q.rbase[owner] + ogt[P.G + age] * q.rstride[owner]];
        const paste_binding bd = pool.bindings[bind];
        const int64_t r = resolve_fast(P.win, pool.steps, bd, bind, ev, age, ogt, memo);
        uint32_t w = 0xffffffffu;
        if (r < 0) {
          atomicOr(q.part + owner, 1ull << ri);
        } else {
          const int64_t osess = warp_first + owner;
          const int64_t node = r & 0xffffffffll;
          const int64_t region =
              n < (1ll << 31) ? (int64_t)((uint32_t)ev / (uint32_t)n) : (int64_t)ev / n;
          if ((int64_t)ev - region * n == osess && region < 31 && node < (1ll << 27))
            w = ((uint32_t)region << 27) | (uint32_t)node;
          else
            ++wide;
        }
        reinterpret_cast<uint32_t*>(stage0 + (size_t)(threadIdx.x - lane + owner) * sstride +
                                    arg_off)[apos] = w;
      }
      count -= take;
      __syncwarp();
    }
  }
  __syncwarp();
  if (!live) return;
  const unsigned long long pm = q.part[lane];
  if (pm) {  // PARTIAL: completeness code and level min(cap, WARM_ONLY)
    for (int i = 0; i < nm; ++i)
      if ((pm >> i) & 1ull) S.pred[i] = (uint16_t)((S.pred[i] & 0x3fff) | (PASTE_C_PARTIAL << 14));
    for (int j = 0; j < n_act; ++j) {
      const int ip = S.act[j] & 31;
      if ((pm >> ip) & 1ull) {
        const int cap = __ldg(P.adm.max_level + __ldg(&recs[ip].tool));
        S.act[j] = (uint8_t)(ip | ((cap < 1 ? cap : 1) << 5));
      }
    }
  }
  c[0] = nm;
  c[1] = na;
  c[2] = n_act;
}

// Write one session's staged records at its stream offsets o[].
__device__ __forceinline__ void compact_flush(const paste_compact_desc& C, int64_t sess,
                                              const Stage& S, const int c[4], const uint64_t o[3],
                                              unsigned long long& wide, uint32_t key) {
  cf_hdr(C, sess, c[0], c[2]);
  if (C.format & PASTE_CF_ENTRY16) {  // the entry key stands for the prediction list
    static_cast<uint16_t*>(C.pred)[sess] = (uint16_t)key;
  } else {
    for (int i = 0; i < c[0]; ++i) {
      const uint16_t v = S.pred[i];
      cf_pred(C, o[0] + i, v & 0x3fff, v >> 14);
    }
  }
  const bool a16 = (C.format & PASTE_CF_ARG16) != 0;
  for (int j = 0; j < c[1]; ++j) {
    const uint32_t w = S.arg[j];
    if (!a16) {
      static_cast<uint32_t*>(C.arg)[o[1] + j] = w;
      continue;
    }
    uint16_t h = 0xffffu;
    if (w != 0xffffffffu) {
      const uint32_t region = w >> 27, node = w & ((1u << 27) - 1);
      if (node < (1u << 11)) h = (uint16_t)((region << 11) | node);
      else ++wide;
    }
    static_cast<uint16_t*>(C.arg)[o[1] + j] = h;
  }
  for (int j = 0; j < c[2]; ++j) C.act[o[2] + j] = S.act[j];
}

__global__ void __launch_bounds__(FT, 8) predict_compact_kernel(const CompactParams Q) {
  extern __shared__ uint64_t s_mem[];
  __shared__ int64_t s_tile;
  __shared__ uint64_t s_warp[FT / 32][4];
  __shared__ uint64_t s_excl[4];
  const FastParams& P = Q.F;
  uint64_t* memo = s_mem;
  for (int i = threadIdx.x; i < MEMO; i += FT) memo[i] = 0;
  int32_t* gt = reinterpret_cast<int32_t*>(s_mem + MEMO) + threadIdx.x * P.row;
  const int K = P.out.max_candidates, B = P.out.max_bindings;
  uint8_t* st = reinterpret_cast<uint8_t*>(s_mem + MEMO) +
                (((size_t)sizeof(int32_t) * FT * P.row + 15) & ~(size_t)15) +
                (size_t)threadIdx.x * stage_stride(K, B);
  const Stage SG{reinterpret_cast<uint16_t*>(st),
                 reinterpret_cast<uint32_t*>(st + ((2 * K + 3) & ~3)),
                 st + ((2 * K + 3) & ~3) + 4 * K * B};
  const int64_t n = P.win.n_sessions;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* stage0 = st - (size_t)threadIdx.x * stage_stride(K, B);
  ResolveQueue* qs = reinterpret_cast<ResolveQueue*>(stage0 + (size_t)FT * stage_stride(K, B));
  int32_t* rows = reinterpret_cast<int32_t*>(s_mem + MEMO) + warp * 32 * P.row;
  unsigned long long wide = 0;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0)
      s_tile = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(Q.ticket), 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= Q.n_tiles) break;
    const int64_t sess = tile * FT + threadIdx.x;
    // ---- the whole step for this session, records staged in shared memory --
    int c[4] = {0, 0, 0, 0};
    uint32_t key = 0xffffu;
    compact_stage(P, sess, sess < n, rows, stage0, stage_stride(K, B), SG, c, memo, qs[warp],
                  wide, key);
    // ---- block-wide exclusive scan of the 4 counters ------------------------
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
    // ---- decoupled look-back (warp 0, 128 predecessor tiles per round) ------
    if (warp == 0) {
      uint64_t agg[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        agg[k] = 0;
        for (int w = 0; w < FT / 32; ++w) agg[k] += s_warp[w][k];
      }
      uint64_t excl[4];
      tile_lookback(Q.tile_state, tile, agg, excl, lane);
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) s_excl[k] = excl[k];
        if (tile == Q.n_tiles - 1) {  // the last tile publishes the totals
          Q.C.totals[0] = (int64_t)(excl[0] + agg[0]);
          Q.C.totals[1] = (int64_t)(excl[1] + agg[1]);
          Q.C.totals[2] = (int64_t)(excl[2] + agg[2]);
          Q.C.totals[4] = (int64_t)(excl[3] + agg[3]);
        }
      }
    }
    __syncthreads();
    if (sess < n) {
      uint64_t o[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        uint64_t before = 0;
        for (int w = 0; w < warp; ++w) before += s_warp[w][k];
        o[k] = s_excl[k] + before + inc[k] - (uint64_t)c[k];
      }
      compact_flush(Q.C, sess, SG, c, o, wide, key);
    }
  }
  if (wide) atomicAdd(reinterpret_cast<unsigned long long*>(Q.C.totals + 3), wide);
}

// Returns true when the fast path handled the launch.
bool predict_fast_dispatch(const paste_pool_desc* pool, const paste_windows* win,
                           const paste_admit_desc* adm, const paste_predict_out* out,
                           int G, cudaStream_t stream) {
  if (G > 16 || out->max_candidates > 32767) return false;
  FastParams P{*pool, *win, *adm, *out, G, 2 * G + 1};
  if (P.pool.match_table != nullptr &&
      (P.pool.mt_k < out->max_candidates || P.pool.mt_g != G || pool->max_bindings > MT_MAX_BIND))
    P.pool.match_table = nullptr;  // stale table: scan instead
  const bool table = P.pool.match_table != nullptr;
  const size_t smem = table && out->max_candidates <= COOP_MAX_K
                          ? coop_smem_bytes(P.row)
                          : sizeof(uint64_t) * MEMO + sizeof(int32_t) * FT * P.row;
  static int sms = 0, per_sm[2] = {0, 0};
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int& occ = per_sm[table ? 1 : 0];
  if (occ == 0) {
    if (table)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, predict_fast_kernel<true>, FT, smem);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, predict_fast_kernel<false>, FT, smem);
    if (occ < 1) occ = 1;
  }
  const int64_t chunks = (win->n_sessions + FT - 1) / FT;
  const int64_t grid = chunks < (int64_t)sms * occ ? chunks : (int64_t)sms * occ;
  if (table)
    predict_fast_kernel<true><<<(unsigned)grid, FT, smem, stream>>>(P);
  else
    predict_fast_kernel<false><<<(unsigned)grid, FT, smem, stream>>>(P);
  return true;
}

// Fused predict + compaction launch; false = not eligible (no match table,
// G > 16, K > 31, ...): the caller runs paste_predict_batch + compaction.
bool compact_eligible(const paste_pool_desc* pool, int K, int B, int format, int G) {
  static const bool force_generic = getenv("PASTE_FORCE_GENERIC") != nullptr;
  if (force_generic || G > 16 || K > 31 || K * B > 64 || pool->match_table == nullptr ||
      pool->mt_k < K || pool->mt_g != G || pool->max_bindings > MT_MAX_BIND ||
      pool->n_patterns > (1 << 14) || ((format & PASTE_CF_HDR8) && K > 15) ||
      ((format & PASTE_CF_PRED8) && pool->n_patterns > 64))
    return false;
  if (format & PASTE_CF_ENTRY16) {  // keys must fit u16 below the 0xFFFF marker
    const int64_t keys = keys_for(pool, G);
    if (keys < 0 || keys >= 0xffff) return false;
  }
  return true;
}

bool predict_compact_dispatch(const paste_pool_desc* pool, const paste_windows* win,
                              const paste_admit_desc* adm, int K, int B,
                              const paste_compact_desc* c, void* scratch, int G,
                              cudaStream_t stream) {
  if (win->stream_end || !compact_eligible(pool, K, B, c->format, G)) return false;
  paste_predict_out out{};
  out.max_candidates = K;
  out.max_bindings = B;
  CompactParams Q{FastParams{*pool, *win, *adm, out, G, 2 * G + 1}, *c,
                  static_cast<uint64_t*>(scratch), static_cast<uint64_t*>(scratch) + LB_STRIDE,
                  (win->n_sessions + FT - 1) / FT};
  const size_t smem = sizeof(uint64_t) * MEMO +
                      (((size_t)sizeof(int32_t) * FT * Q.F.row + 15) & ~(size_t)15) +
                      (size_t)FT * stage_stride(K, B) + sizeof(ResolveQueue) * (FT / 32);
  static int sms = 0, occ = 0, occ_smem = 0;
  cudaFuncSetAttribute(predict_compact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       96 * 1024);  // per device context: every call
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (occ_smem != (int)smem) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, predict_compact_kernel, FT, smem);
    if (occ < 1) occ = 1;
    occ_smem = (int)smem;
  }
  const int64_t grid = Q.n_tiles < (int64_t)sms * occ ? Q.n_tiles : (int64_t)sms * occ;
  predict_compact_kernel<<<(unsigned)grid, FT, smem, stream>>>(Q);
  return true;
}

}  // namespace paste

extern "C" int paste_predict_compact_supported(const paste_pool_desc* pool,
                                               int32_t window_capacity, int32_t max_candidates,
                                               int32_t max_bindings, int32_t format) {
  using namespace paste;
  if (!pool || window_capacity < 1 || max_candidates < 1 || max_bindings < pool->max_bindings)
    return 0;
  return compact_eligible(pool, max_candidates, max_bindings, format,
                          gather_depth(pool, window_capacity))
             ? 1
             : 0;
}

extern "C" int64_t paste_predict_compact_scratch_bytes(int64_t n_sessions) {
  const int64_t tiles = (n_sessions + paste::FT - 1) / paste::FT;
  return 8 * (paste::LB_STRIDE * tiles + paste::LB_STRIDE);
}

extern "C" int paste_predict_compact(const paste_pool_desc* pool, paste_windows* windows,
                                     const paste_admit_desc* admit, int32_t max_candidates,
                                     int32_t max_bindings, paste_compact_desc* out, void* scratch,
                                     void* stream) {
  using namespace paste;
  reset_launches();
  PASTE_REQUIRE(pool && windows && admit && out && scratch, "null argument");
  PASTE_REQUIRE(windows->capacity >= 1 && max_candidates >= 1, "bad window / candidate count");
  PASTE_REQUIRE(max_bindings >= pool->max_bindings, "max_bindings below pool maximum");
  PASTE_REQUIRE(!windows->stream_end, "stream-mode windows are not live sessions");
  PASTE_REQUIRE(!windows->new_tok8 && !windows->new_node16 && !windows->new_node8 && !(out->format & PASTE_CF_KEYS),
                "narrow observe form / PASTE_CF_KEYS need paste_predict_live_compact");
  cudaStream_t st = (cudaStream_t)stream;
  PASTE_CUDA_CHECK(cudaMemsetAsync(scratch, 0, paste_predict_compact_scratch_bytes(windows->n_sessions), st));
  PASTE_CUDA_CHECK(cudaMemsetAsync(out->totals, 0, 5 * sizeof(int64_t), st));
  if (windows->n_sessions == 0) return PASTE_OK;
  const int g = pool->relation == PASTE_REL_ANCHORED ? pool->k : pool->max_ctx;
  const int G = g < windows->capacity ? g : windows->capacity;
  static const bool force_generic = getenv("PASTE_FORCE_GENERIC") != nullptr;
  if (force_generic || !predict_compact_dispatch(pool, windows, admit, max_candidates,
                                                 max_bindings, out, scratch, G, st)) {
    set_error("fused predict + compaction needs the match-table fast path (K <= 31, "
              "<= 16384 patterns): use paste_predict_batch + paste_compact_records");
    return PASTE_ERR_UNSUPPORTED;
  }
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
