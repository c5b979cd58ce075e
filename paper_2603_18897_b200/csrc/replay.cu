// C2 replay: score_accuracy (prediction.py:133-169) as two launches.
//
//   1. K4 (paste_predict_batch) predicts every window, reading it in place
//      from the event stream (paste_windows stream mode: the `call_len`
//      events before each call);
//   2. replay_score_kernel: one thread per call tallies top1 / top3 and the
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
#include "fast.cuh"

namespace paste {

__device__ __forceinline__ uint32_t lower4(uint32_t y) {  // ASCII A-Z -> a-z, bytewise
  const uint32_t up = __vcmpgeu4(y, 0x41414141u) & __vcmpleu4(y, 0x5a5a5a5au);
  return y + (up & 0x20202020u);
}

// a == lower(b) over n ASCII bytes (str.lower on ASCII text), 8 bytes a step
__device__ __forceinline__ bool bytes_eq_lower(const uint8_t* a, const uint8_t* b, int64_t n) {
  for (int64_t k = 0; k < n; k += 8) {
    const int r = n - k < 8 ? (int)(n - k) : 8;
    const uint64_t y = ld_part8(b + k, r);
    const uint64_t ly = (uint64_t)lower4((uint32_t)y) | ((uint64_t)lower4((uint32_t)(y >> 32)) << 32);
    if (ld_part8(a + k, r) != ly) return false;
  }
  return true;
}

__device__ __forceinline__ bool bytes_ascii(const uint8_t* a, int64_t n) {
  uint64_t acc = 0;
  for (int64_t k = 0; k < n; k += 8) acc |= ld_part8(a + k, n - k < 8 ? (int)(n - k) : 8);
  return (acc & 0x8080808080808080ull) == 0;
}

__device__ __forceinline__ bool node_ascii(const Node& nd, const uint8_t* b, int64_t n) {
  return (nd.flags() & PASTE_F_ASCII) || bytes_ascii(b, n);
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
  int64_t al = 0;
  const uint8_t* ab = at < PASTE_T_LIST ? canon_bytes(D, a, ar.byte_base, &al) : nullptr;
  if (kind != PASTE_X_FORMAT) {
    const int pt = pn.type();
    if (pt >= PASTE_T_LIST || at >= PASTE_T_LIST) return pt == at ? CMP_UNSURE : CMP_NE;
    if (pt != at) return CMP_NE;
    if (pt <= PASTE_T_TRUE) return CMP_EQ;
    int64_t pl;
    const uint8_t* pb = canon_bytes(D, pn, pr.byte_base, &pl);
    if (pt == PASTE_T_STR && !((pn.flags() & a.flags()) & PASTE_F_ASCII) &&
        (has_surrogate(pb, pl) || has_surrogate(ab, al)))
      return CMP_UNSURE;  // json.dumps(...).encode("utf-8") raises on lone surrogates
    return (pl == al && bytes_eq(pb, ab, pl)) ? CMP_EQ : CMP_NE;
  }
  // FormatTemplate: prefix + norm(leaf_str(leaf)) + suffix (mappings.py:197-223)
  if (at != PASTE_T_STR) return CMP_NE;
  const uint8_t* tb = D.bytes + pr.byte_base + pn.a;  // leaf_str: raw text / number text
  int64_t lo = 0, hi = pn.b;
  const int* f = D.fmt + 5 * bind;
  const int pl = f[1], sl = f[3], norm = f[4] & 0xff;
  if ((f[4] & PASTE_FMT_NON_ASCII) || !node_ascii(pn, tb, hi) || !node_ascii(a, ab, al))
    return CMP_UNSURE;  // Unicode str.strip / str.lower / NFC: the host decides
  const uint8_t* pre = D.fmt_bytes + f[0];
  const uint8_t* suf = D.fmt_bytes + f[2];
  if (norm == 1) {  // str.strip()
    while (lo < hi && py_space_ascii(tb[lo])) ++lo;
    while (hi > lo && py_space_ascii(tb[hi - 1])) --hi;
  }
  if ((int64_t)pl + (hi - lo) + sl != al) return CMP_NE;
  if (!bytes_eq(pre, ab, pl)) return CMP_NE;
  if (!(norm == 2 ? bytes_eq_lower(ab + pl, tb + lo, hi - lo) : bytes_eq(ab + pl, tb + lo, hi - lo)))
    return CMP_NE;
  return bytes_eq(suf, ab + pl + (hi - lo), sl) ? CMP_EQ : CMP_NE;
}

__device__ __forceinline__ int64_t lookup_key(const paste_tape_node* nodes, int64_t base,
                                              int32_t key) {
  return step_child(nodes, base, 0, 0, key);
}

// Verdict of candidate i of call c (a FULL candidate of the call's tool with
// the call's key set): every binding's value must equal the argument.
__device__ __forceinline__ int candidate_verdict(const paste_pool_desc& pool,
                                                 const paste_replay_desc& D,
                                                 const paste_predict_out& out, int64_t c, int i) {
  const int64_t n = D.n_calls;
  const int32_t pid = out.pred_pat[out_at(out, n, c, i)];
  const paste_pattern pat = pool.patterns[pid];
  const int nb = (pat.flags & PASTE_PF_HAS_MAPPING) ? pat.n_bind : 0;
  const int32_t aev = D.call_args[c];
  const int64_t abase = D.refs[aev].node_base;
  int verdict = CMP_EQ;
  for (int b = 0; b < nb && verdict != CMP_NE; ++b) {
    const int bind = pat.bind_off + b;
    const int64_t pref = out.pred_arg[arg_at(out, n, c, i, b)];
    const int64_t an = lookup_key(D.nodes, abase, D.bind_key[bind]);
    if (pref < 0 || an < 0) {  // cannot happen for FULL + equal key sets; stay exact
      verdict = CMP_UNSURE;
      continue;
    }
    const int r = compare_binding(D, bind, pool.bindings[bind].kind, pref, aev, an);
    if (r == CMP_NE) verdict = CMP_NE;
    else if (r == CMP_UNSURE) verdict = CMP_UNSURE;
  }
  return verdict;
}

// One warp scores 32 calls (lane = call) per iteration.  The cheap part --
// top1 / top3 and the key-set filter -- runs lane per call; the candidates that
// need argument comparison go through a per-warp queue in shared memory and
// are compared one candidate per lane, so lanes stay busy however unevenly
// the comparisons fall over the calls (a lane-per-call loop ran ~6 of 32
// lanes active).  Verdicts land in per-warp bit masks (bit = call lane).
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_CHUNK = 8;  // candidate records loaded per round

__global__ void __launch_bounds__(RS_THREADS, 4) replay_score_kernel(const paste_pool_desc pool,
                                                                  const paste_replay_desc D,
                                                                  const paste_predict_out out) {
  __shared__ uint16_t queue[RS_WARPS][32 + RS_CHUNK * 32];
  __shared__ unsigned hit_mask[RS_WARPS], unsure_mask[RS_WARPS];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t n = D.n_calls;
  const int64_t stride = (int64_t)gridDim.x * RS_WARPS * 32;
  unsigned long long c1 = 0, c3 = 0, ch = 0, cu = 0;
  for (int64_t base = ((int64_t)blockIdx.x * RS_WARPS + w) * 32; base < n; base += stride) {
    const int64_t c = base + lane;
    const bool live = c < n;
    int np = 0;
    int32_t tool = -1, cks = -2;
    if (live) {
      np = out.n_pred[c];
      const int lim = D.cand_limit;
      np = lim >= 0 ? (np < lim ? np : lim) : (np + lim > 0 ? np + lim : 0);
      tool = D.call_tool[c];
      cks = D.call_keyset[c];
    }
    if (lane == 0) {
      hit_mask[w] = 0u;
      unsure_mask[w] = 0u;
    }
    __syncwarp();
    bool top1 = false, top3 = false, unsure = false;
    int count = 0;
    const int max_np = __reduce_max_sync(FULL, (unsigned)np);
    for (int i0 = 0; i0 < max_np; i0 += RS_CHUNK) {
      // issue the chunk's record loads together (independent, slot-major rows)
      int32_t pidv[RS_CHUNK];
      uint8_t compv[RS_CHUNK];
#pragma unroll
      for (int j = 0; j < RS_CHUNK; ++j) {
        pidv[j] = 0;
        compv[j] = 0xff;
        if (i0 + j < np) {
          const int64_t o = out_at(out, n, c, i0 + j);
          pidv[j] = out.pred_pat[o];
          compv[j] = out.pred_comp[o];
        }
      }
#pragma unroll
      for (int j = 0; j < RS_CHUNK; ++j) {
        const int i = i0 + j;
        bool need = false;
        if (i < np) {
          const bool same = __ldg(&pool.patterns[pidv[j]].target_tool) == tool;
          if (i == 0) top1 = same;
          if (i < 3) top3 |= same;
          if (same && compv[j] == PASTE_C_FULL && cks != -2) {  // -2: args not a dict
            const int32_t pks = __ldg(D.pat_keyset + pidv[j]);
            if (pks < 0 || cks < 0) unsure = true;
            else need = pks == cks;
          }
        }
        const unsigned m = __ballot_sync(FULL, need);
        if (need) queue[w][count + __popc(m & lt)] = (uint16_t)((lane << 8) | i);
        count += __popc(m);
      }
      __syncwarp();
      // drain full rounds of 32 (one queued candidate per lane); after the
      // last chunk also the remainder.  Newest entries first, so the kept
      // ones stay at the front of the queue.
      const bool last = i0 + RS_CHUNK >= max_np;
      while (count >= 32 || (last && count > 0)) {
        const int take = count < 32 ? count : 32;
        if (lane < take) {
          const uint16_t it = queue[w][count - take + lane];
          const int src = it >> 8;
          const int v = candidate_verdict(pool, D, out, base + src, it & 0xff);
          if (v == CMP_EQ) atomicOr(&hit_mask[w], 1u << src);
          else if (v == CMP_UNSURE) atomicOr(&unsure_mask[w], 1u << src);
        }
        count -= take;
        __syncwarp();
      }
    }
    __syncwarp();
    if (live) {
      const bool hit = (hit_mask[w] >> lane) & 1u;
      unsure = (unsure || ((unsure_mask[w] >> lane) & 1u)) && !hit;
      D.unsure[c] = unsure;
      c1 += top1;
      c3 += top3;
      ch += hit;
      cu += unsure;
    }
    __syncwarp();
  }
  // block reduction, one atomic per counter per block
  __shared__ unsigned long long red[4][RS_WARPS];
  for (int off = 16; off; off >>= 1) {
    c1 += __shfl_down_sync(FULL, c1, off);
    c3 += __shfl_down_sync(FULL, c3, off);
    ch += __shfl_down_sync(FULL, ch, off);
    cu += __shfl_down_sync(FULL, cu, off);
  }
  if (lane == 0) {
    red[0][w] = c1;
    red[1][w] = c3;
    red[2][w] = ch;
    red[3][w] = cu;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    unsigned long long s = 0;
    for (int k = 0; k < RS_WARPS; ++k) s += red[threadIdx.x][k];
    if (s) atomicAdd(reinterpret_cast<unsigned long long*>(D.tallies) + threadIdx.x, s);
  }
}

// ---------------------------------------------------------------------------
// Fused replay: windows -> match-table candidates -> score, one kernel, no
// prediction records.  Scoring needs far less than the records: top1 / top3
// are the target tools of the first three table records; a hit needs a FULL
// candidate of the call's tool with the call's key set, so only those
// candidates' bindings are resolved (resolve_fast, the K4 walk) and compared
// (compare_binding) -- every other candidate is never resolved.  FULL = every
// binding resolves; a candidate with an unresolved binding cannot hit.
// Calls the device cannot decide (Unicode / containers / key sets the host
// interns as -1) are flagged exactly as replay_score_kernel flags them.
// ---------------------------------------------------------------------------
constexpr int RF_THREADS = 256;
constexpr int RF_WARPS = RF_THREADS / 32;
constexpr int RF_GMAX = 8;
constexpr int RF_CHUNK = 8;
constexpr int RF_PEEK = 6;  // window events gathered in one batch

__global__ void __launch_bounds__(RF_THREADS, 4) replay_fused_kernel(const paste_pool_desc pool,
                                                                   const paste_replay_desc D,
                                                                   int K, int G) {
  __shared__ int32_t gts[RF_WARPS][32][2 * RF_GMAX];  // gathered tokens, then event ids
  __shared__ const uint8_t* ents[RF_WARPS][32];
  __shared__ uint32_t queue[RF_WARPS][32 + RF_CHUNK * 32];
  __shared__ unsigned hit_mask[RF_WARPS], unsure_mask[RF_WARPS];
  __shared__ int32_t s_aev[RF_WARPS][32];   // the call's actual-argument payload
  __shared__ int64_t s_abase[RF_WARPS][32];  // and its node base
  __shared__ uint64_t memo[MEMO];
  for (int i = threadIdx.x; i < MEMO; i += RF_THREADS) memo[i] = 0;
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t n = D.n_calls;
  const int S = pool.n_bucket_sigs;
  const int64_t stride = (int64_t)gridDim.x * RF_WARPS * 32;
  const int64_t mts = mt_stride(pool.mt_k);
  paste_windows win{};
  win.nodes = D.nodes;
  win.bytes = D.bytes;
  win.refs = const_cast<paste_event_ref*>(D.refs);
  unsigned long long c1 = 0, c3 = 0, ch = 0, cu = 0;
  for (int64_t base = ((int64_t)blockIdx.x * RF_WARPS + w) * 32; base < n; base += stride) {
    const int64_t c = base + lane;
    const bool live = c < n;
    int32_t* gt = gts[w][lane];
    int32_t* ge = gt + RF_GMAX;
    // ---- gather the newest G tool events of the call's window ---------------
    int m = 0;
    int32_t tool = -1, cks = -2;
    if (live) {
      const int64_t end = D.call_pos[c];
      const int64_t lo = end - D.call_len[c];
      tool = D.call_tool[c];
      cks = D.call_keyset[c];
      const int32_t aev = D.call_args[c];
      s_aev[w][lane] = aev;
      // the newest RF_PEEK events in one batch of independent loads (a
      // window's newest G tool events are almost always among them)
      const int span = end - lo < RF_PEEK ? (int)(end - lo) : RF_PEEK;
      int32_t tk[RF_PEEK], ev[RF_PEEK];
#pragma unroll
      for (int j = 0; j < RF_PEEK; ++j) {
        tk[j] = j < span ? __ldg(D.ev_tok + end - 1 - j) : -1;
        ev[j] = j < span ? __ldg(D.ev_evt + end - 1 - j) : -1;
      }
      s_abase[w][lane] = aev >= 0 ? D.refs[aev].node_base : 0;
#pragma unroll
      for (int j = 0; j < RF_PEEK; ++j)
        if (tk[j] >= 0 && m < G) {
          gt[m] = tk[j];
          ge[m] = ev[j];
          ++m;
        }
      for (int64_t q = end - 1 - span; q >= lo && m < G; --q) {  // longer LLM runs
        const int32_t t = __ldg(D.ev_tok + q);
        if (t >= 0) {
          gt[m] = t;
          ge[m] = __ldg(D.ev_evt + q);
          ++m;
        }
      }
    }
    const uint8_t* e = nullptr;
    int np = 0;
    if (live && m > 0 && gt[0] < S) {
      int64_t key = gt[0], mult = S;
      for (int a = 1; a < G; ++a) {
        const int t = a < m ? gt[a] : S;
        key += (int64_t)(t < S ? t : S) * mult;
        mult *= (S + 1);
      }
      e = static_cast<const uint8_t*>(pool.match_table) + key * mts;
      const int nm0 = __ldg(reinterpret_cast<const int*>(e));
      const int nm = nm0 < K ? nm0 : K;
      const int lim = D.cand_limit;
      np = lim >= 0 ? (nm < lim ? nm : lim) : (nm + lim > 0 ? nm + lim : 0);
    }
    ents[w][lane] = e;
    if (lane == 0) {
      hit_mask[w] = 0u;
      unsure_mask[w] = 0u;
    }
    __syncwarp();
    bool top1 = false, top3 = false;
    int count = 0;
    const int max_np = __reduce_max_sync(FULL, (unsigned)np);
    for (int i0 = 0; i0 < max_np; i0 += RF_CHUNK) {
      int4 rv[RF_CHUNK];
#pragma unroll
      for (int j = 0; j < RF_CHUNK; ++j)
        rv[j] = i0 + j < np ? __ldg(reinterpret_cast<const int4*>(e + 16 + 32 * (i0 + j)))
                            : make_int4(0, 0, -1, 0);
#pragma unroll
      for (int j = 0; j < RF_CHUNK; ++j) {
        const int i = i0 + j;
        uint32_t item = 0;
        bool need = false;
        if (i < np) {
          const bool same = rv[j].z == tool;
          if (i == 0) top1 = same;
          if (i < 3) top3 |= same;
          if (same && ((rv[j].w >> 16) & PASTE_PF_HAS_MAPPING) && cks != -2) {
            const int32_t pks = __ldg(D.pat_keyset + rv[j].x);
            if (pks < 0 || cks < 0) {
              need = true;  // undecided key sets: unsure iff the candidate is FULL
              item = 1u << 15;
            } else {
              need = pks == cks;
            }
          }
        }
        const unsigned msk = __ballot_sync(FULL, need);
        if (need) queue[w][count + __popc(msk & lt)] = ((uint32_t)lane << 16) | item | (uint32_t)i;
        count += __popc(msk);
      }
      __syncwarp();
      const bool last = i0 + RF_CHUNK >= max_np;
      while (count >= 32 || (last && count > 0)) {
        const int take = count < 32 ? count : 32;
        if (lane < take) {
          const uint32_t it = queue[w][count - take + lane];
          const int src = it >> 16, i = it & 0x7fff;
          const bool ks_unsure = (it >> 15) & 1u;
          const int4 r0 = __ldg(reinterpret_cast<const int4*>(ents[w][src] + 16 + 32 * i));
          const int4 r1 = __ldg(reinterpret_cast<const int4*>(ents[w][src] + 16 + 32 * i) + 1);
          const uint32_t ages = (uint32_t)r0.y;
          const int n_bind = r0.w & 0xffff, bind_off = r1.x;
          const int32_t* ogt = gts[w][src];
          const int32_t* oge = ogt + RF_GMAX;
          const int32_t aev = s_aev[w][src];
          const int64_t abase = s_abase[w][src];
          int verdict = CMP_EQ;
          for (int b = 0; b < n_bind; ++b) {
            const int bind = bind_off + b;
            const paste_binding bd = pool.bindings[bind];
            const int age = (ages >> (4 * b)) & 15;
            const int64_t r = resolve_fast(win, pool.steps, bd, bind, oge[age], age, ogt, memo);
            if (r < 0) {  // PARTIAL: not a hit candidate
              verdict = CMP_NE;
              break;
            }
            if (ks_unsure) {
              verdict = CMP_UNSURE;
              continue;
            }
            const int64_t an = lookup_key(D.nodes, abase, D.bind_key[bind]);
            const int v = an < 0 ? CMP_UNSURE : compare_binding(D, bind, bd.kind, r, aev, an);
            if (v == CMP_NE) {
              verdict = CMP_NE;
              break;
            }
            if (v == CMP_UNSURE) verdict = CMP_UNSURE;
          }
          if (verdict == CMP_EQ) atomicOr(&hit_mask[w], 1u << src);
          else if (verdict == CMP_UNSURE) atomicOr(&unsure_mask[w], 1u << src);
        }
        count -= take;
        __syncwarp();
      }
    }
    __syncwarp();
    if (live) {
      const bool hit = (hit_mask[w] >> lane) & 1u;
      const bool unsure = ((unsure_mask[w] >> lane) & 1u) && !hit;
      D.unsure[c] = unsure;
      c1 += top1;
      c3 += top3;
      ch += hit;
      cu += unsure;
    }
    __syncwarp();
  }
  __shared__ unsigned long long red[4][RF_WARPS];
  for (int off = 16; off; off >>= 1) {
    c1 += __shfl_down_sync(FULL, c1, off);
    c3 += __shfl_down_sync(FULL, c3, off);
    ch += __shfl_down_sync(FULL, ch, off);
    cu += __shfl_down_sync(FULL, cu, off);
  }
  if (lane == 0) {
    red[0][w] = c1;
    red[1][w] = c3;
    red[2][w] = ch;
    red[3][w] = cu;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    unsigned long long s = 0;
    for (int k = 0; k < RF_WARPS; ++k) s += red[threadIdx.x][k];
    if (s) atomicAdd(reinterpret_cast<unsigned long long*>(D.tallies) + threadIdx.x, s);
  }
}

}  // namespace paste

using namespace paste;

extern "C" int paste_replay_fused(const paste_pool_desc* pool, const paste_replay_desc* d,
                                  int32_t max_candidates, void* stream) {
  reset_launches();
  PASTE_REQUIRE(pool && d, "null descriptor");
  PASTE_REQUIRE(d->capacity >= 1, "window capacity must be >= 1");
  PASTE_REQUIRE(max_candidates >= 1, "max_candidates must be >= 1");
  const int G = pool->mt_g;
  if (!pool->match_table || pool->mt_k < max_candidates || G < 1 || G > RF_GMAX ||
      pool->max_bindings > 8) {
    set_error("pool / window outside the fused replay envelope (needs a match table)");
    return PASTE_ERR_UNSUPPORTED;
  }
  if (d->n_calls == 0) return PASTE_OK;
  // one resident wave (a second partial wave left most warps idle at the end)
  static int resident = 0;
  if (resident == 0) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, replay_fused_kernel, RF_THREADS, 0);
    resident = sms * (occ > 0 ? occ : 1);
  }
  int64_t blocks = (d->n_calls + RF_THREADS - 1) / RF_THREADS;
  if (blocks > resident) blocks = resident;
  replay_fused_kernel<<<(unsigned)blocks, RF_THREADS, 0, (cudaStream_t)stream>>>(
      *pool, *d, max_candidates, G);
  PASTE_CUDA_CHECK(cudaGetLastError());
  count_launch(1);
  return PASTE_OK;
}

extern "C" int paste_replay_score(const paste_pool_desc* pool, const paste_replay_desc* d,
                                  paste_predict_out* out, void* stream) {
  reset_launches();
  PASTE_REQUIRE(pool && d && out, "null descriptor");
  PASTE_REQUIRE(d->capacity >= 1, "window capacity must be >= 1");
  if (d->n_calls == 0) return PASTE_OK;
  const cudaStream_t st = (cudaStream_t)stream;
  paste_windows win{};
  win.n_sessions = d->n_calls;
  win.capacity = d->capacity;
  win.tok = const_cast<int32_t*>(d->ev_tok);  // read-only in stream mode
  win.evt = const_cast<int32_t*>(d->ev_evt);
  win.count = const_cast<int64_t*>(d->call_len);
  win.stream_end = d->call_pos;
  win.nodes = d->nodes;
  win.bytes = d->bytes;
  win.refs = const_cast<paste_event_ref*>(d->refs);
  PASTE_REQUIRE(out->max_candidates <= 256, "replay supports at most 256 candidates per call");
  paste_admit_desc adm{};
  const int rc = paste_predict_batch(pool, &win, &adm, out, stream);
  if (rc != PASTE_OK) return rc;
  int64_t blocks = (d->n_calls + RS_THREADS - 1) / RS_THREADS;
  if (blocks > 148 * 8) blocks = 148 * 8;
  replay_score_kernel<<<(unsigned)blocks, RS_THREADS, 0, st>>>(*pool, *d, *out);
  PASTE_CUDA_CHECK(cudaGetLastError());
  count_launch(1);  // + the K4 launches counted by paste_predict_batch
  return PASTE_OK;
}
