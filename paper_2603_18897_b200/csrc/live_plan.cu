// Live plan: the live step (K4 / the serving step) with everything that
// depends only on the match-table key precomputed.
//
// Reference: PredictionWindow.observe + Predictor.predict + admit
// (prediction.py:40-118, mining.py:119-156, mappings.py:143-223,
// policy.py:207-244), one session per tool completion (simulation.py:402-442).
//
// Which patterns match, their rank order, which bindings must be resolved
// (and against which matched event), and the admit decisions -- which
// candidate wins each tool, its level when the prediction is complete, its
// utility p * benefit -- all depend only on the newest G tool tokens (the
// match-table key) and the per-tool admit tables: admission does not depend
// on completeness, only the level does (a PARTIAL prediction is admitted at
// min(cap, WARM_ONLY)).  paste_build_live_plan therefore compiles, per key,
// the step's records; the live kernel per session is
//
//   observe (ring write, directory entry)  ->  newest G-1 older tool tokens
//   (one batch of independent loads)  ->  key  ->  plan entry (L1/L2)  ->
//   copy the records, resolve the entry's bindings (walk table: the resolved
//   node of a PathLookup / FormatTemplate binding depends only on (binding,
//   node array), one L1/L2 load), downgrade PARTIAL predictions.
//
// Each thread runs SPT sessions (j * FT + thread of a tile) with their loads
// interleaved, for memory-level parallelism.  The serving form writes the
// narrow streams directly: stream counts depend only on the key, so a tile
// publishes its aggregate (decoupled look-back) before any binding is
// resolved, and every record is written once at its final offset -- no
// staging.
#include <cooperative_groups.h>
#include <string.h>

#include <type_traits>

#include "common.cuh"

namespace paste {

constexpr int LT = 128;  // threads per CTA

__host__ __device__ inline int plan_align(int x, int a) { return (x + a - 1) / a * a; }

struct PlanLayout {
  int K, M;                  // candidate slots, binding slots (K * max_bindings)
  int off_pid, off_comp, off_act, off_util, off_map;
  int64_t stride;
};

__host__ __device__ inline PlanLayout plan_layout(int K, int max_bind) {
  PlanLayout L;
  L.K = K;
  L.M = K * (max_bind > 0 ? max_bind : 1);
  L.off_pid = 16;
  L.off_comp = L.off_pid + 4 * K;
  L.off_act = plan_align(L.off_comp + K, 16);
  L.off_util = plan_align(L.off_act + 2 * K, 8);
  L.off_map = L.off_util + 8 * K;
  L.stride = plan_align(L.off_map + 8 * L.M, 16);
  return L;
}

struct MTRec {  // the match-table record (predict_fast.cu, 32 bytes)
  int32_t pid;
  uint32_t src;
  int32_t tool;
  int32_t nb_flags;
  int32_t bind_off;
  int32_t pad;
  double p;
};

// true when bindings a and b resolve to the same node of the same source
// payload (the caller compares the source ages): same expression kind and
// the same path steps (and, for IndexedFallback, the same suffix, start
// index and fail tool).  ctx_pos is not compared -- the age stands for it.
__device__ inline bool same_resolution(const paste_pool_desc& pool, int a, int b) {
  if (a == b) return true;
  const paste_binding x = pool.bindings[a], y = pool.bindings[b];
  if (x.kind != y.kind || x.step_cnt != y.step_cnt) return false;
  const bool fb = x.kind == PASTE_X_FALLBACK;
  if (fb && (x.suf_cnt != y.suf_cnt || x.start_index != y.start_index ||
             x.fail_tool != y.fail_tool))
    return false;
  const int2* st = reinterpret_cast<const int2*>(pool.steps);
  for (int i = 0; i < x.step_cnt; ++i) {
    const int2 u = st[x.step_off + i], v = st[y.step_off + i];
    if (u.x != v.x || u.y != v.y) return false;
  }
  if (fb)
    for (int i = 0; i < x.suf_cnt; ++i) {
      const int2 u = st[x.suf_off + i], v = st[y.suf_off + i];
      if (u.x != v.x || u.y != v.y) return false;
    }
  return true;
}

// one thread per key: admit the key's first K matches exactly as admit()
// does (policy.py:207-244) and lay the records out.  Map word q:
// binding | rank << 32 | bslot << 40 | source age << 48 | unit << 56, where
// the units number the entry's distinct resolutions (same_resolution at the
// same age) in first-use order; duplicates only ever point at units < 64.
__global__ void build_live_plan_kernel(const paste_pool_desc pool, const paste_admit_desc adm,
                                       const uint8_t* table, int64_t mt_stride, int64_t n_keys,
                                       PlanLayout L, uint8_t* plan) {
  const int64_t key = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (key >= n_keys) return;
  const uint8_t* e = table + key * mt_stride;
  const int32_t* hdr = reinterpret_cast<const int32_t*>(e);
  const MTRec* rec = reinterpret_cast<const MTRec*>(e + 16);
  uint8_t* P = plan + key * L.stride;
  const int nm = hdr[0] < L.K ? hdr[0] : L.K;
  int32_t* pid = reinterpret_cast<int32_t*>(P + L.off_pid);
  uint8_t* comp = P + L.off_comp;
  uint16_t* act = reinterpret_cast<uint16_t*>(P + L.off_act);
  double* util = reinterpret_cast<double*>(P + L.off_util);
  uint64_t* map = reinterpret_cast<uint64_t*>(P + L.off_map);
  int n_act = 0, n_map = 0;
  for (int i = 0; i < nm; ++i) {
    const MTRec r = rec[i];
    const int flags = r.nb_flags >> 16, nb = r.nb_flags & 0xffff;
    const bool mapped = (flags & PASTE_PF_HAS_MAPPING) != 0;
    const int c = mapped ? PASTE_C_FULL : PASTE_C_TOOL_ONLY;
    pid[i] = r.pid;
    comp[i] = (uint8_t)c;
    if (mapped)
      for (int b = 0; b < nb && n_map < L.M; ++b)
        map[n_map++] = (uint64_t)(uint32_t)(r.bind_off + b) | ((uint64_t)i << 32) |
                       ((uint64_t)b << 40) | ((uint64_t)((r.src >> (4 * b)) & 15u) << 48);
    if (!adm.enabled || r.tool >= adm.n_tools || !adm.allow[r.tool]) continue;
    const int cap = adm.max_level[r.tool];
    const int implied = c == PASTE_C_FULL ? 3 : 1;
    const int lv_full = cap < implied ? cap : implied, lv_part = cap < 1 ? cap : 1;
    const uint16_t a = (uint16_t)(i | (lv_full << 8) | (lv_part << 12));
    const double u = __dmul_rn(r.p, adm.benefit[r.tool]);
    int j = 0;  // the tool's incumbent (first-appearance order is kept)
    for (; j < n_act; ++j)
      if (rec[act[j] & 0xff].tool == r.tool) break;
    if (j == n_act) {
      act[n_act] = a;
      util[n_act] = u;
      ++n_act;
      continue;
    }
    const double iu = util[j], ip = rec[act[j] & 0xff].p;
    if ((u != iu) ? (u > iu) : (r.p > ip)) {  // _beats: (utility, p, -created_at)
      act[j] = a;
      util[j] = u;
    }
  }
  int n_unit = 0;
  for (int q = 0; q < n_map; ++q) {
    const int bq = (int)(uint32_t)map[q], aq = (int)((map[q] >> 48) & 0xff);
    int u = -1;
    for (int p = 0; p < q && u < 0; ++p) {
      const int up = (int)(map[p] >> 56);
      if (up < 64 && (int)((map[p] >> 48) & 0xff) == aq && same_resolution(pool, (int)(uint32_t)map[p], bq))
        u = up;
    }
    if (u < 0) u = n_unit++;
    map[q] |= (uint64_t)u << 56;
  }
  P[0] = (uint8_t)nm;
  P[1] = (uint8_t)n_act;
  P[2] = (uint8_t)n_map;
  P[3] = (uint8_t)n_unit;
  reinterpret_cast<int32_t*>(P)[1] = hdr[1];
}

// one thread per (binding, node): the node a PathLookup / FormatTemplate
// binding resolves to in the payload whose tape starts at `node`; -1 =
// unresolved, -2 = resolve at run time (IndexedFallback counts failures)
__global__ void build_walk_kernel(const paste_pool_desc pool, int32_t n_bind,
                                  const paste_tape_node* nodes, int64_t n_nodes, int32_t* walk) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n_bind * n_nodes) return;
  const int64_t bind = i / n_nodes, base = i - bind * n_nodes;
  const paste_binding bd = pool.bindings[bind];
  if (bd.kind == PASTE_X_FALLBACK) {
    walk[i] = -2;
    return;
  }
  int64_t cur = 0;
  const int2* st = reinterpret_cast<const int2*>(pool.steps);
  for (int s = 0; s < bd.step_cnt && cur >= 0; ++s) {
    const int2 k = st[bd.step_off + s];
    cur = step_child(nodes, base, cur, k.x, k.y);
  }
  if (bd.kind == PASTE_X_FORMAT && cur >= 0) {  // _leaf_str holes (mappings.py:197-204)
    const int t = load_node(nodes, base + cur).type();
    if (t != PASTE_T_STR && t != PASTE_T_INT && t != PASTE_T_FLOAT) cur = -1;
  }
  walk[i] = cur >= 0 && cur < (1ll << 31) ? (int32_t)cur : -1;
}


// ---------------------------------------------------------------------------
// the live kernel
// ---------------------------------------------------------------------------
struct LiveParams {
  paste_pool_desc pool;
  paste_windows win;
  paste_predict_out out;  // K-slot records (predict form)
  paste_compact_desc C;   // narrow streams (serving form)
  const uint8_t* plan;
  PlanLayout L;
  const int32_t* walk;
  int64_t walk_nodes;
  int admit;
  int S;                  // n_bucket_sigs
  int fast8;              // K = 8, slot-major, n * K * B < 2^31 (kslot_write8)
  // two-pass serving form: per-session staging (session-major, L2-resident)
  int32_t* st_key;        // [n] match-table key, -1 = none
  uint32_t* st_cnt;       // [n] nm | n_act << 5 | n_map << 10 | n_err << 18
  uint32_t* st_part;      // [n] PARTIAL mask
  uint32_t* st_arg;       // [n][M] encoded argument words (stream width applied later)
  int M;
  // key-stream form: per-warp argument counts and exclusive offsets
  uint32_t* w_cnt;
  uint64_t* ticket;
  uint64_t* tile_state;
  int64_t n_tiles;
};

template <int G>
struct Sess {
  int64_t s;
  int32_t ev0;             // the observed event
  int64_t node0;           // its node base
  int newest;              // ring slot of the observed event, -1 = it is not a tool event
  uint32_t slots;          // ring slot (< 16) of the tool event of age a at bits 4a
  int32_t tk[G];           // newest tool tokens by age
  int m;
  const uint8_t* e;        // plan entry (nullptr = no predictions)
  int32_t key;             // match-table key, -1 = none
  int nm, n_act, n_err;
  int n_map;               // map entries | distinct units << 8 (the plan header)
};

// ring addressing of session s (derived, not kept per session: registers)
__device__ __forceinline__ int64_t ring_base(const LiveParams& P, int64_t s) {
  return P.win.slot_major ? s : s * P.win.capacity;
}
__device__ __forceinline__ int64_t ring_stride(const LiveParams& P) {
  return P.win.slot_major ? P.win.n_sessions : 1;
}

// newest G tool tokens: the G-1 older ring slots in one batch of loads; an
// LLM step (-1) among them falls back to the slot-by-slot scan
template <int G>
__device__ __forceinline__ void gather_slow(const LiveParams& P, Sess<G>& x, int32_t t_new,
                                            int len, int head) {
  const int W = P.win.capacity;
  x.m = 0;
  x.slots = 0;
  int slot = head;
  for (int i = 0; i < len && x.m < G; ++i) {
    const int32_t t = i == 0 ? t_new : P.win.tok[ring_base(P, x.s) + slot * ring_stride(P)];
    if (t >= 0) {
#pragma unroll
      for (int q = 0; q < G; ++q)
        if (q == x.m) x.tk[q] = t;
      x.slots |= (uint32_t)slot << (4 * x.m);
      ++x.m;
    }
    slot = slot == 0 ? W - 1 : slot - 1;
  }
}

// stage 1: the session's inputs (independent loads; the values are not
// consumed here, so the loads stay in flight across a pipelined round)
struct FrontIn {
  int64_t s, cnt;
  paste_event_ref ref;  // new_ref form
  int32_t node;         // new_node form
  int32_t t;
};

__device__ __forceinline__ void front_load(const LiveParams& P, int64_t s, FrontIn& f) {
  f.s = s;
  if (s >= P.win.n_sessions) return;
  f.cnt = P.win.count[s];
  if (P.win.new_tok8 != nullptr) {  // narrow wire form: u8 token, u16 node or u8 node code
    f.t = P.win.new_tok8[s];         // (or the u8 event code alone: event_codes)
    f.node = P.win.new_node8 != nullptr    ? (int32_t)P.win.new_node8[s]
             : P.win.new_node16 != nullptr ? (int32_t)P.win.new_node16[s]
                                           : 0;
    return;
  }
  f.t = P.win.new_tok[s];
  if (P.win.new_node != nullptr)
    f.node = P.win.new_node[s];
  else
    f.ref = P.win.new_ref[s];
}

__device__ __forceinline__ int wrap_sub(int a, int b, int W) {  // (a - b) mod W, 0 <= a, b < W
  const int d = a - b;
  return d < 0 ? d + W : d;
}

// stage 2: observe (ring slot, directory entry, count) and issue the loads of
// the G-1 older ring slots
template <int G>
struct FrontMid {
  int32_t ot[G > 1 ? G - 1 : 1];
  int32_t t_new;
  int len;
};

template <int G>
__device__ __forceinline__ void front_observe(const LiveParams& P, const FrontIn& f, Sess<G>& y,
                                              FrontMid<G>& m) {
  const int64_t n = P.win.n_sessions;
  const int W = P.win.capacity;
  y.s = f.s;
  y.e = nullptr;
  y.key = -1;
  y.nm = y.n_act = y.n_map = y.n_err = 0;
  if (f.s >= n) return;
  const int64_t rbase = ring_base(P, f.s), rstride = ring_stride(P);
  int32_t t_in = (P.win.new_tok8 != nullptr && f.t == 255) ? -1 : f.t;
  int32_t node_in = f.node;
  if (P.win.event_codes != nullptr) {  // 1-byte form: u8 event code -> (token, node_base)
    const int2 e = __ldg(reinterpret_cast<const int2*>(P.win.event_codes) + f.t);
    t_in = e.x;
    node_in = e.y;
  }
  const int head = (W & (W - 1)) == 0 ? (int)(f.cnt & (W - 1))
                   : f.cnt < (1ll << 31) ? (int)((uint32_t)f.cnt % (uint32_t)W)
                                         : (int)(f.cnt % W);
  y.ev0 = (int32_t)(P.win.new_evt_base + f.s);
  const bool narrow = P.win.new_node != nullptr || P.win.new_tok8 != nullptr;
  y.node0 = narrow ? (int64_t)(P.win.new_node8 != nullptr ? __ldg(P.win.node_codes + f.node) : node_in)
                   : f.ref.node_base;
  P.win.refs[y.ev0] =
      paste_event_ref{y.node0, (narrow ? 0 : f.ref.byte_base) + P.win.new_byte_base};
  P.win.tok[rbase + head * rstride] = t_in;
  P.win.evt[rbase + head * rstride] = y.ev0;
  const int64_t c1 = f.cnt + 1;
  P.win.count[f.s] = c1;
  y.newest = head;
  m.t_new = t_in;
  m.len = (int)(c1 < W ? c1 : W);
#pragma unroll
  for (int a = 1; a < G; ++a) {
    m.ot[a - 1] = -1;
    if (a < m.len) m.ot[a - 1] = P.win.tok[rbase + wrap_sub(head, a, W) * rstride];
  }
}

// stage 3: the newest G tool tokens, the key and the plan entry header
template <int G, bool COMPACT>
__device__ __forceinline__ void front_key(const LiveParams& P, Sess<G>& y, const FrontMid<G>& m) {
  if (y.s >= P.win.n_sessions) return;
  const int W = P.win.capacity;
  bool fast = m.t_new >= 0;
  y.tk[0] = m.t_new;
  y.slots = (uint32_t)y.newest;
  y.m = 1;
#pragma unroll
  for (int a = 1; a < G; ++a) {
    if (a < m.len) {
      fast = fast && m.ot[a - 1] >= 0;
      y.tk[a] = m.ot[a - 1];
      y.slots |= (uint32_t)wrap_sub(y.newest, a, W) << (4 * a);
      y.m = a + 1;
    }
  }
  if (!fast) {
    gather_slow<G>(P, y, m.t_new, m.len, y.newest);
    if (m.t_new < 0) y.newest = -1;
  }
  if (y.m > 0 && y.tk[0] < P.S) {
    int key = y.tk[0], mult = P.S;  // keys < 2^31 (paste_live_plan_bytes)
#pragma unroll
    for (int a = 1; a < G; ++a) {
      const int t = a < y.m ? y.tk[a] : P.S;
      key += (t < P.S ? t : P.S) * mult;
      mult *= P.S + 1;
    }
    y.e = P.plan + (int64_t)key * P.L.stride;
    y.key = key;
    const int2 h = *reinterpret_cast<const int2*>(y.e);
    y.nm = h.x & 0xff;
    y.n_act = (h.x >> 8) & 0xff;
    y.n_map = (h.x >> 16) & 0xffff;
    y.n_err = h.y;
  }
}

template <int G, int SPT, bool COMPACT>
__device__ __forceinline__ void live_front(const LiveParams& P, int64_t base, Sess<G> (&x)[SPT]) {
  FrontIn f[SPT];
  FrontMid<G> m[SPT];
#pragma unroll
  for (int j = 0; j < SPT; ++j) front_load(P, base + j * LT + threadIdx.x, f[j]);
#pragma unroll
  for (int j = 0; j < SPT; ++j) front_observe<G>(P, f[j], x[j], m[j]);
#pragma unroll
  for (int j = 0; j < SPT; ++j) front_key<G, COMPACT>(P, x[j], m[j]);
}

// resolve the entry's bindings for session y; returns the PARTIAL mask and
// calls emit(rank, bslot, ev, node) for every binding (node < 0 =
// unresolved).  With `units` (PASTE_CF_UNIQ) a binding whose resolution
// unit was already resolved is not resolved or emitted again: it takes the
// unit's outcome for the PARTIAL mask, and emit runs once per unit.
template <int G, typename F>
__device__ __forceinline__ uint32_t live_resolve(const LiveParams& P, const Sess<G>& y, F emit,
                                                 bool units = false) {
  uint32_t part = 0;
  uint64_t bad = 0;  // unresolved units (< 64)
  int nu = 0;
  const uint64_t* map = reinterpret_cast<const uint64_t*>(y.e + P.L.off_map);
  const int n_map = y.n_map & 0xff;
  for (int q = 0; q < n_map; ++q) {
    const uint64_t w = map[q];
    const int bind = (int)(uint32_t)w, rank = (int)((w >> 32) & 0xff), bslot = (int)((w >> 40) & 0xff);
    const int age = (int)((w >> 48) & 0xff), unit = (int)(w >> 56);
    if (units) {
      if (unit < nu) {  // a repeat of an earlier unit
        if (unit < 64 && ((bad >> unit) & 1ull)) part |= 1u << rank;
        continue;
      }
      ++nu;
    }
    const int slot = (int)((y.slots >> (4 * age)) & 15);
    int32_t ev;
    int64_t nb;
    if (slot == y.newest) {
      ev = y.ev0;
      nb = y.node0;
    } else {
      ev = P.win.evt[ring_base(P, y.s) + slot * ring_stride(P)];
      nb = P.win.refs[ev].node_base;
    }
    int64_t cur = -2;
    if (P.walk != nullptr && nb >= 0 && nb < P.walk_nodes) cur = P.walk[(int64_t)bind * P.walk_nodes + nb];
    if (cur == -2) {  // IndexedFallback, or outside the walk table
      const paste_binding bd = P.pool.bindings[bind];
      int fails = 0;  // FAIL events of fail_tool after the source (mappings.py:185-194)
      if (bd.kind == PASTE_X_FALLBACK) {
#pragma unroll
        for (int a = 0; a < G; ++a)
          if (a < age) fails += ((y.tk[a] >> 1) == bd.fail_tool) && ((y.tk[a] & 1) == 0);
      }
      cur = walk_binding(P.win, P.pool.steps, bd, nb, fails);
    }
    if (cur < 0) {
      part |= 1u << rank;
      if (units && unit < 64) bad |= 1ull << unit;
    }
    emit(rank, bslot, ev, cur);
  }
  return part;
}

// true when any lane of this lane's aligned group of g lanes has its bit in
// `mask` (g = 32-byte sector / element size): a store that only some lanes
// of a sector make is a partial-sector write, which L2 completes with a DRAM
// read; filling the sector's other slots with don't-care values avoids it
__device__ __forceinline__ bool group_any(unsigned mask, int g) {
  const int lane = threadIdx.x & 31;
  if (g >= 32) return mask != 0;
  const unsigned gm = ((1u << g) - 1u) << (lane & ~(g - 1));
  return (mask & gm) != 0;
}

// K-slot records of one session from its plan entry (called by every active
// lane of the warp together).  Slots past n_pred / n_act (and unmapped
// argument slots) are don't-care; in slot-major layout the lanes write them
// wherever a neighbour's record shares the 32-byte sector, so every sector is
// written whole.
template <int G>
__device__ __forceinline__ void kslot_write(const LiveParams& P, const Sess<G>& y) {
  const int64_t n = P.win.n_sessions;
  const int K = P.out.max_candidates, B = P.out.max_bindings;
  const bool sm = P.out.slot_major != 0;
  const int64_t ostride = sm ? n : 1;
  const int64_t obase = sm ? y.s : y.s * K;
  const int64_t abase = sm ? y.s : y.s * K * B;
  const unsigned act_m = __activemask();
  uint32_t part = 0;
  uint64_t mapped = 0;  // (rank * B + bslot) bits of the written arguments
  if (y.n_map > 0)
    part = live_resolve<G>(P, y, [&](int rank, int bslot, int32_t ev, int64_t cur) {
      P.out.pred_arg[abase + (int64_t)(rank * B + bslot) * ostride] =
          cur < 0 ? -1 : (((int64_t)ev << 32) | cur);
      mapped |= 1ull << ((rank * B + bslot) & 63);
    });
  const int max_nm = (int)__reduce_max_sync(act_m, (unsigned)y.nm);
  const int max_na = (int)__reduce_max_sync(act_m, (unsigned)y.n_act);
  const int4* pid4 = reinterpret_cast<const int4*>(y.e + P.L.off_pid);
  const uint32_t* comp4 = reinterpret_cast<const uint32_t*>(y.e + P.L.off_comp);
  int32_t* pp = P.out.pred_pat + obase;
  uint8_t* pc = P.out.pred_comp + obase;
  for (int i0 = 0; i0 < max_nm; i0 += 4) {
    int4 v = make_int4(-1, -1, -1, -1);
    uint32_t cw = 0;
    if (i0 < y.nm) {
      v = pid4[i0 >> 2];
      cw = comp4[i0 >> 2];
    }
    const int pv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u;
      if (i >= max_nm) break;
      const bool mine = i < y.nm;
      const unsigned have = __ballot_sync(act_m, mine);
      if (mine || (sm && group_any(have, 8))) pp[i * ostride] = mine ? pv[u] : -1;
      if (mine || (sm && have)) {
        const uint8_t c = ((part >> i) & 1u) ? (uint8_t)PASTE_C_PARTIAL : (uint8_t)(cw >> (8 * u));
        pc[i * ostride] = mine ? c : (uint8_t)PASTE_C_TOOL_ONLY;
      }
    }
  }
  if (sm && K * B <= 64) {  // unmapped argument slots that share a sector with a written one
    uint64_t pairs = mapped;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pairs |= __shfl_xor_sync(act_m, pairs, o);
    while (pairs) {
      const int bit = __ffsll((long long)pairs) - 1;
      pairs &= pairs - 1;
      const unsigned have = __ballot_sync(act_m, (mapped >> bit) & 1ull);
      if (!((mapped >> bit) & 1ull) && group_any(have, 4))
        P.out.pred_arg[abase + (int64_t)bit * ostride] = -1;
    }
  }
  if (max_na > 0) {
    const uint16_t* act = reinterpret_cast<const uint16_t*>(y.e + P.L.off_act);
    const double* util = reinterpret_cast<const double*>(y.e + P.L.off_util);
    for (int a = 0; a < max_na; ++a) {
      const bool mine = a < y.n_act;
      const unsigned have = __ballot_sync(act_m, mine);
      const int64_t o = obase + a * ostride;
      uint16_t v = 0;
      double u = 0.0;
      if (mine) {
        v = act[a];
        u = util[a];
      }
      const int slot = v & 0xff;
      if (mine || (sm && group_any(have, 16))) P.out.act_pred[o] = (int16_t)(mine ? slot : -1);
      if (mine || (sm && have))
        P.out.act_level[o] = (uint8_t)(((part >> slot) & 1u) ? (v >> 12) & 15 : (v >> 8) & 15);
      if (mine || (sm && group_any(have, 4))) P.out.act_util[o] = u;
    }
  }
  P.out.n_pred[y.s] = y.nm;
  P.out.struct_err[y.s] = y.n_err;
  if (P.admit) P.out.n_act[y.s] = y.n_act;
}

// max of v over this lane's aligned group of g lanes (full warp only)
template <int g>
__device__ __forceinline__ int group_max(int v) {
#pragma unroll
  for (int o = 1; o < g; o <<= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// K = 8, slot-major, full warp: the same records with the sector fill
// computed once per quantity (group maxima over the 8 / 16 / 4 / 32 lanes
// that share a 32-byte sector of a 4 / 2 / 8 / 1-byte array) and 32-bit
// record offsets.  Argument slots are written only where resolved.
template <int G>
__device__ __forceinline__ void kslot_write8(const LiveParams& P, const Sess<G>& y) {
  const uint32_t n = (uint32_t)P.win.n_sessions;
  const uint32_t s = (uint32_t)y.s;
  const int B = P.out.max_bindings;
  uint32_t part = 0;
  if (y.n_map > 0)
    part = live_resolve<G>(P, y, [&](int rank, int bslot, int32_t ev, int64_t cur) {
      P.out.pred_arg[(uint32_t)(rank * B + bslot) * n + s] =
          cur < 0 ? -1 : (((int64_t)ev << 32) | cur);
    });
  const int nm = y.nm, na = y.n_act;
  const int nm8 = group_max<8>(nm);
  const int nm32 = max(nm8, __shfl_xor_sync(0xffffffffu, max(nm8, __shfl_xor_sync(0xffffffffu, nm8, 8)), 16));
  const int na4 = group_max<4>(na);
  int na_16 = max(na4, __shfl_xor_sync(0xffffffffu, na4, 4));
  na_16 = max(na_16, __shfl_xor_sync(0xffffffffu, na_16, 8));
  const int na32 = max(na_16, __shfl_xor_sync(0xffffffffu, na_16, 16));
  int4 p0 = make_int4(-1, -1, -1, -1), p1 = p0;
  uint64_t cw = 0x0202020202020202ull;  // TOOL_ONLY
  uint4 av = make_uint4(0, 0, 0, 0);
  if (y.e) {
    p0 = *reinterpret_cast<const int4*>(y.e + P.L.off_pid);
    p1 = *reinterpret_cast<const int4*>(y.e + P.L.off_pid + 16);
    cw = *reinterpret_cast<const uint64_t*>(y.e + P.L.off_comp);
    av = *reinterpret_cast<const uint4*>(y.e + P.L.off_act);
  }
  const int pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
  const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
  const double* util = reinterpret_cast<const double*>(y.e + P.L.off_util);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t o = (uint32_t)i * n + s;
    const bool mine = i < nm;
    if (i < nm8) P.out.pred_pat[o] = mine ? pv[i] : -1;
    if (i < nm32)
      P.out.pred_comp[o] = !mine ? (uint8_t)PASTE_C_TOOL_ONLY
                           : ((part >> i) & 1u) ? (uint8_t)PASTE_C_PARTIAL
                                                : (uint8_t)(cw >> (8 * i));
  }
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    if (a >= na32) break;
    const uint32_t o = (uint32_t)a * n + s;
    const bool mine = a < na;
    const uint32_t v = (aw[a >> 1] >> (16 * (a & 1))) & 0xffffu;
    const int slot = (int)(v & 0xff);
    if (a < na_16) P.out.act_pred[o] = (int16_t)(mine ? slot : -1);
    P.out.act_level[o] = (uint8_t)(((part >> slot) & 1u) ? (v >> 12) & 15 : (v >> 8) & 15);
    if (a < na4) P.out.act_util[o] = mine ? util[a] : 0.0;
  }
  P.out.n_pred[s] = nm;
  P.out.struct_err[s] = y.n_err;
  if (P.admit) P.out.n_act[s] = na;
}

// Persistent CTAs, one session per thread per round, software-pipelined over
// rounds: round r+2's inputs and round r+1's older ring slots are in flight
// while round r is keyed and written, so the count -> ring -> plan chain
// costs one memory round trip per round instead of three.
template <int G, int MINB = 7>
__global__ void __launch_bounds__(LT, MINB) predict_live_kernel(const LiveParams P) {
  const int64_t n = P.win.n_sessions;
  const int64_t stride = (int64_t)gridDim.x * LT;
  const int64_t s0 = (int64_t)blockIdx.x * LT + threadIdx.x;
  FrontIn f1, f2;
  Sess<G> y0, y1;
  FrontMid<G> m0, m1;
  front_load(P, s0, f1);
  front_load(P, s0 + stride, f2);
  front_observe<G>(P, f1, y1, m1);
  for (int64_t s = s0; s < n; s += stride) {
    y0 = y1;
    m0 = m1;
    f1 = f2;
    front_load(P, s + 2 * stride, f2);
    front_observe<G>(P, f1, y1, m1);
    front_key<G, false>(P, y0, m0);
    if (P.fast8 && __activemask() == 0xffffffffu)
      kslot_write8<G>(P, y0);
    else
      kslot_write<G>(P, y0);
  }
}

// block-wide exclusive offsets of the 4 stream counters in session order
// (j-major within the tile), with a decoupled look-back across tiles
template <int SPT>
__device__ __forceinline__ void live_offsets(const LiveParams& P, int64_t tile, const int c[SPT][4],
                                             uint64_t off[SPT][4]) {
  __shared__ uint32_t s_w[SPT][LT / 32][4];
  __shared__ uint64_t s_ex[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc[SPT][4];
#pragma unroll
  for (int j = 0; j < SPT; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t v = (uint32_t)c[j][k];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      inc[j][k] = v;
      if (lane == 31) s_w[j][warp][k] = v;
    }
  __syncthreads();
  if (warp == 0) {
    uint64_t agg[4], ex[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      agg[k] = 0;
      for (int j = 0; j < SPT; ++j)
        for (int w = 0; w < LT / 32; ++w) agg[k] += s_w[j][w][k];
    }
    tile_lookback(P.tile_state, tile, agg, ex, lane);
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) s_ex[k] = ex[k];
      if (tile == P.n_tiles - 1) {
        P.C.totals[0] = (int64_t)(ex[0] + agg[0]);
        P.C.totals[1] = (int64_t)(ex[1] + agg[1]);
        P.C.totals[2] = (int64_t)(ex[2] + agg[2]);
        P.C.totals[4] = (int64_t)(ex[3] + agg[3]);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint64_t run = s_ex[k];
#pragma unroll
    for (int j = 0; j < SPT; ++j) {
      uint64_t before = 0, all = 0;
      for (int w = 0; w < LT / 32; ++w) {
        all += s_w[j][w][k];
        if (w < warp) before += s_w[j][w][k];
      }
      off[j][k] = run + before + inc[j][k] - (uint32_t)c[j][k];
      run += all;
    }
  }
}

// the session's key-stream element: the u16 match-table key, or with
// PASTE_CF_KEY8 the entry's u8 plan code (header byte 8); all-ones = none
template <int G>
__device__ __forceinline__ void key_write(const paste_compact_desc& C, const Sess<G>& y) {
  if (C.format & PASTE_CF_KEY8)
    static_cast<uint8_t*>(C.pred)[y.s] = y.key >= 0 ? y.e[8] : (uint8_t)0xffu;
  else
    static_cast<uint16_t*>(C.pred)[y.s] = y.key >= 0 ? (uint16_t)y.key : (uint16_t)0xffffu;
}

// argument words a session writes: one per binding, or one per resolution
// unit (PASTE_CF_UNIQ); none without predictions
template <int G>
__device__ __forceinline__ int arg_count(const LiveParams& P, const Sess<G>& y) {
  if (y.nm == 0) return 0;
  return (P.C.format & PASTE_CF_UNIQ) ? (y.n_map >> 8) & 0xff : y.n_map & 0xff;
}

// one session's records in the narrow streams at its offsets off[4]
template <int G>
__device__ __forceinline__ void compact_write(const LiveParams& P, const Sess<G>& y,
                                              const uint64_t off[4], unsigned long long& wide) {
  const int64_t n = P.win.n_sessions;
  const paste_compact_desc& C = P.C;
  const bool a16 = (C.format & PASTE_CF_ARG16) != 0;
  const bool keys = (C.format & PASTE_CF_KEYS) != 0;
  const bool units = (C.format & PASTE_CF_UNIQ) != 0;
  if (!keys) cf_hdr(C, y.s, y.nm, y.n_act);
  uint32_t part = 0;
  if (y.nm > 0 && y.n_map > 0) {
    int q = 0;
    const uint64_t oa = off[1];
    part = live_resolve<G>(P, y, [&](int, int, int32_t ev, int64_t cur) {
      uint32_t w = a16 ? 0xffffu : 0xffffffffu;
      if (cur >= 0) {
        const int64_t region =
            n < (1ll << 31) ? (int64_t)((uint32_t)ev / (uint32_t)n) : (int64_t)ev / n;
        if ((int64_t)ev - region * n == y.s && region < 31 && cur < (a16 ? (1ll << 11) : (1ll << 27)))
          w = a16 ? (((uint32_t)region << 11) | (uint32_t)cur)
                  : (((uint32_t)region << 27) | (uint32_t)cur);
        else
          ++wide;
      }
      if (a16) static_cast<uint16_t*>(C.arg)[oa + q] = (uint16_t)w;
      else static_cast<uint32_t*>(C.arg)[oa + q] = w;
      ++q;
    }, units);
  }
  if (C.format & PASTE_CF_ENTRY16) {
    key_write<G>(C, y);
  } else if (y.nm > 0) {
    const int32_t* pid = reinterpret_cast<const int32_t*>(y.e + P.L.off_pid);
    const uint8_t* comp = y.e + P.L.off_comp;
    for (int i = 0; i < y.nm; ++i)
      cf_pred(C, off[0] + i, pid[i], ((part >> i) & 1u) ? PASTE_C_PARTIAL : comp[i]);
  }
  if (y.n_act > 0 && !keys) {
    const uint16_t* act = reinterpret_cast<const uint16_t*>(y.e + P.L.off_act);
    for (int a = 0; a < y.n_act; ++a) {
      const uint16_t v = act[a];
      const int slot = v & 0xff;
      const int lv = ((part >> slot) & 1u) ? (v >> 12) & 15 : (v >> 8) & 15;
      C.act[off[2] + a] = (uint8_t)(slot | (lv << 5));
    }
  }
}

// tiles claimed through a ticket (SPT sessions per thread)
template <int G, int SPT>
__global__ void __launch_bounds__(LT) predict_live_compact_kernel(const LiveParams P) {
  __shared__ int64_t s_tile;
  const int64_t n = P.win.n_sessions;
  unsigned long long wide = 0;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0)
      s_tile = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(P.ticket), 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= P.n_tiles) break;
    Sess<G> x[SPT];
    live_front<G, SPT, true>(P, tile * LT * SPT, x);
    int c[SPT][4];
#pragma unroll
    for (int j = 0; j < SPT; ++j) {
      c[j][0] = x[j].nm;
      c[j][1] = arg_count(P, x[j]);
      c[j][2] = x[j].n_act;
      c[j][3] = x[j].n_err;
    }
    uint64_t off[SPT][4];
    live_offsets<SPT>(P, tile, c, off);
#pragma unroll
    for (int j = 0; j < SPT; ++j)
      if (x[j].s < n) compact_write<G>(P, x[j], off[j], wide);
  }
  if (wide) atomicAdd(reinterpret_cast<unsigned long long*>(P.C.totals + 3), wide);
}

// ---- two-pass serving form ---------------------------------------------
// Pass 1 is predict_live_kernel's pipelined step writing, per session, the
// fixed-position streams (hdr, and the ENTRY16 key) plus a staging record
// (key, counts, PARTIAL mask, resolved argument words) that stays in L2.
// Pass 2 scans the counts (decoupled look-back over light tiles) and
// scatters the variable-length streams.  The step itself thus runs without
// any cross-CTA wait; only the light scatter does.
template <int G>
__device__ __forceinline__ void stage_write(const LiveParams& P, const Sess<G>& y,
                                            unsigned long long& wide) {
  const int64_t n = P.win.n_sessions;
  const paste_compact_desc& C = P.C;
  const bool a16 = (C.format & PASTE_CF_ARG16) != 0;
  uint32_t part = 0;
  int q = 0;  // argument words staged
  if (y.nm > 0 && y.n_map > 0) {
    uint32_t* sa = P.st_arg + y.s * P.M;
    part = live_resolve<G>(P, y, [&](int, int, int32_t ev, int64_t cur) {
      uint32_t w = a16 ? 0xffffu : 0xffffffffu;
      if (cur >= 0) {
        const int64_t region =
            n < (1ll << 31) ? (int64_t)((uint32_t)ev / (uint32_t)n) : (int64_t)ev / n;
        if ((int64_t)ev - region * n == y.s && region < 31 && cur < (a16 ? (1ll << 11) : (1ll << 27)))
          w = a16 ? (((uint32_t)region << 11) | (uint32_t)cur)
                  : (((uint32_t)region << 27) | (uint32_t)cur);
        else
          ++wide;
      }
      sa[q++] = w;
    }, (C.format & PASTE_CF_UNIQ) != 0);
  }
  if (!(C.format & PASTE_CF_KEYS)) cf_hdr(C, y.s, y.nm, y.n_act);
  if (C.format & PASTE_CF_ENTRY16)
    key_write<G>(C, y);
  P.st_key[y.s] = y.key;
  P.st_cnt[y.s] = (uint32_t)y.nm | ((uint32_t)y.n_act << 5) | ((uint32_t)q << 10) |
                  ((uint32_t)y.n_err << 18);
  P.st_part[y.s] = part;
}

template <int G>
__global__ void __launch_bounds__(LT) predict_live_stage_kernel(const LiveParams P) {
  const int64_t n = P.win.n_sessions;
  const int64_t stride = (int64_t)gridDim.x * LT;
  const int64_t s0 = (int64_t)blockIdx.x * LT + threadIdx.x;
  unsigned long long wide = 0;
  FrontIn f1, f2;
  Sess<G> y0, y1;
  FrontMid<G> m0, m1;
  front_load(P, s0, f1);
  front_load(P, s0 + stride, f2);
  front_observe<G>(P, f1, y1, m1);
  for (int64_t s = s0; s < n; s += stride) {
    y0 = y1;
    m0 = m1;
    f1 = f2;
    front_load(P, s + 2 * stride, f2);
    front_observe<G>(P, f1, y1, m1);
    front_key<G, false>(P, y0, m0);
    stage_write<G>(P, y0, wide);
  }
  if (wide) atomicAdd(reinterpret_cast<unsigned long long*>(P.C.totals + 3), wide);
}

constexpr int SCAT_SPT = 4;

// ---- key-stream serving form (PASTE_CF_KEYS) ----------------------------
// With the key stream only the argument stream has a variable length, and a
// session's argument count follows from its key.  The step writes each
// warp's argument words (32 consecutive sessions) contiguously into the
// warp's staging slot (capacity 32 * M) at the warp-exclusive offsets, and
// the warp's total; a copy kernel scans the warp totals (tiles of 256
// warps, decoupled look-back over ~120 tiles per 1M sessions) and moves
// every warp's words to their final offset.  No barrier in the step.
struct KeyTotals {  // per thread (32-bit: a thread runs few sessions; registers are tight)
  uint32_t nm, na, ne, wide;
};

template <int G>
__device__ __forceinline__ void keys_write(const LiveParams& P, const Sess<G>& y, KeyTotals& t) {
  const int64_t n = P.win.n_sessions;
  const paste_compact_desc& C = P.C;
  const int lane = threadIdx.x & 31;
  const bool live = y.s < n;
  const int cnt = live ? arg_count(P, y) : 0;
  int inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  const int64_t w = (y.s - lane) >> 5;  // warp base is a multiple of 32
  if (lane == 31) P.w_cnt[w] = (uint32_t)inc;
  if (!live) return;
  const bool a16 = (C.format & PASTE_CF_ARG16) != 0;
  if (cnt > 0) {
    const int64_t at = w * 32 * P.M + (inc - cnt);
    int q = 0;
    live_resolve<G>(P, y, [&](int, int, int32_t ev, int64_t cur) {
      uint32_t wd = a16 ? 0xffffu : 0xffffffffu;
      if (cur >= 0) {
        const int64_t region =
            n < (1ll << 31) ? (int64_t)((uint32_t)ev / (uint32_t)n) : (int64_t)ev / n;
        if ((int64_t)ev - region * n == y.s && region < 31 && cur < (a16 ? (1ll << 11) : (1ll << 27)))
          wd = a16 ? (((uint32_t)region << 11) | (uint32_t)cur)
                   : (((uint32_t)region << 27) | (uint32_t)cur);
        else
          ++t.wide;
      }
      if (a16) reinterpret_cast<uint16_t*>(P.st_arg)[at + q] = (uint16_t)wd;
      else P.st_arg[at + q] = wd;
      ++q;
    }, (C.format & PASTE_CF_UNIQ) != 0);
  }
  key_write<G>(C, y);
  t.nm += (unsigned)y.nm;
  t.na += (unsigned)y.n_act;
  t.ne += (unsigned)y.n_err;
}

template <int G, int MINB>
__global__ void __launch_bounds__(LT, MINB) predict_live_keys_kernel(const LiveParams P) {
  const int64_t n = P.win.n_sessions;
  const int64_t stride = (int64_t)gridDim.x * LT;
  const int64_t s0 = (int64_t)blockIdx.x * LT + threadIdx.x;
  const int lane = threadIdx.x & 31;
  {  // the copy kernel's ticket and tile records (it runs after this kernel)
    const int64_t words = LB_STRIDE * (P.n_tiles + 1);
    for (int64_t i = (int64_t)blockIdx.x * LT + threadIdx.x; i < words; i += stride)
      P.ticket[i] = 0;
  }
  KeyTotals t{0, 0, 0, 0};
  FrontIn f1, f2;
  Sess<G> y0, y1;
  FrontMid<G> m0, m1;
  front_load(P, s0, f1);
  front_load(P, s0 + stride, f2);
  front_observe<G>(P, f1, y1, m1);
  for (int64_t s = s0; s - lane < n; s += stride) {  // warp-uniform: whole warps
    y0 = y1;
    m0 = m1;
    f1 = f2;
    front_load(P, s + 2 * stride, f2);
    front_observe<G>(P, f1, y1, m1);
    front_key<G, false>(P, y0, m0);
    keys_write<G>(P, y0, t);
  }
  {
    const unsigned long long nm = __reduce_add_sync(0xffffffffu, t.nm);
    const unsigned long long na = __reduce_add_sync(0xffffffffu, t.na);
    const unsigned long long ne = __reduce_add_sync(0xffffffffu, t.ne);
    const unsigned long long wd = __reduce_add_sync(0xffffffffu, t.wide);
    if (lane == 0) {
      unsigned long long* tot = reinterpret_cast<unsigned long long*>(P.C.totals);
      if (nm) atomicAdd(tot + 0, nm);
      if (na) atomicAdd(tot + 2, na);
      if (wd) atomicAdd(tot + 3, wd);
      if (ne) atomicAdd(tot + 4, ne);
    }
  }
}

// The key-stream step, the warp-total scan and the copy in ONE cooperative
// kernel (every CTA resident): after the pipelined step a grid barrier; CTA
// b then sums the warp totals of its contiguous range of staged warps; a
// second barrier; each CTA adds up the sums of the CTAs before it, scans its
// range and copies those warps' words to their final offset.  Two grid
// barriers instead of two more launches.
template <int G, int MINB>
__global__ void __launch_bounds__(LT, MINB) predict_live_keys_coop_kernel(const LiveParams P) {
  namespace cg = cooperative_groups;
  const int64_t n = P.win.n_sessions;
  const int64_t stride = (int64_t)gridDim.x * LT;
  const int64_t s0 = (int64_t)blockIdx.x * LT + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  KeyTotals t{0, 0, 0, 0};
  {
    FrontIn f1, f2;
    Sess<G> y0, y1;
    FrontMid<G> m0, m1;
    front_load(P, s0, f1);
    front_load(P, s0 + stride, f2);
    front_observe<G>(P, f1, y1, m1);
    for (int64_t s = s0; s - lane < n; s += stride) {  // warp-uniform: whole warps
      y0 = y1;
      m0 = m1;
      f1 = f2;
      front_load(P, s + 2 * stride, f2);
      front_observe<G>(P, f1, y1, m1);
      front_key<G, false>(P, y0, m0);
      keys_write<G>(P, y0, t);
    }
  }
  {
    const unsigned long long nm = __reduce_add_sync(0xffffffffu, t.nm);
    const unsigned long long na = __reduce_add_sync(0xffffffffu, t.na);
    const unsigned long long ne = __reduce_add_sync(0xffffffffu, t.ne);
    const unsigned long long wd = __reduce_add_sync(0xffffffffu, t.wide);
    if (lane == 0) {
      unsigned long long* tot = reinterpret_cast<unsigned long long*>(P.C.totals);
      if (nm) atomicAdd(tot + 0, nm);
      if (na) atomicAdd(tot + 2, na);
      if (wd) atomicAdd(tot + 3, wd);
      if (ne) atomicAdd(tot + 4, ne);
    }
  }
  cg::grid_group grid = cg::this_grid();
  __threadfence();
  grid.sync();  // every warp total is written
  __shared__ uint64_t s_red[LT / 32];
  __shared__ uint64_t s_base;
  const int64_t nw = (n + 31) / 32;
  const int64_t per = (nw + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = (int64_t)blockIdx.x * per;
  const int64_t w1 = w0 + per < nw ? w0 + per : nw;
  uint64_t* cta_sum = P.tile_state;  // [gridDim.x]
  uint64_t part = 0;
  for (int64_t w = w0 + threadIdx.x; w < w1; w += LT) part += P.w_cnt[w];
  part = __reduce_add_sync(0xffffffffu, (unsigned)part);
  if (lane == 0) s_red[warp] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t v = 0;
    for (int k = 0; k < LT / 32; ++k) v += s_red[k];
    cta_sum[blockIdx.x] = v;
  }
  __threadfence();
  grid.sync();  // every CTA's sum is written
  uint64_t before = 0;
  for (int64_t b = threadIdx.x; b < blockIdx.x; b += LT) before += cta_sum[b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
  __syncthreads();
  if (lane == 0) s_red[warp] = before;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t v = 0;
    for (int k = 0; k < LT / 32; ++k) v += s_red[k];
    s_base = v;
    if (blockIdx.x == gridDim.x - 1) P.C.totals[1] = (int64_t)(v + cta_sum[blockIdx.x]);
  }
  __syncthreads();
  // scan the range LT warps at a time, then copy: staged warp w goes to warp
  // (w - chunk) % (LT / 32) of this CTA, lanes copy its words
  __shared__ uint32_t s_c[LT], s_o[LT];
  uint64_t run = s_base;
  const bool a16 = (P.C.format & PASTE_CF_ARG16) != 0;
  for (int64_t c0 = w0; c0 < w1; c0 += LT) {
    const int64_t w = c0 + threadIdx.x;
    const uint32_t c = w < w1 ? P.w_cnt[w] : 0u;
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) s_red[warp] = inc;
    __syncthreads();
    uint64_t wb = 0, all = 0;
    for (int k = 0; k < LT / 32; ++k) {
      if (k < warp) wb += s_red[k];
      all += s_red[k];
    }
    s_c[threadIdx.x] = c;
    s_o[threadIdx.x] = (uint32_t)(run + wb + inc - c);
    __syncthreads();
    const int nk = (int)(w1 - c0 < LT ? w1 - c0 : LT);
    for (int j = warp; j < nk; j += LT / 32) {
      const uint32_t cj = s_c[j], oj = s_o[j];
      const int64_t src = (c0 + j) * 32 * P.M;
      for (uint32_t i = lane; i < cj; i += 32) {
        if (a16)
          static_cast<uint16_t*>(P.C.arg)[oj + i] = reinterpret_cast<const uint16_t*>(P.st_arg)[src + i];
        else
          static_cast<uint32_t*>(P.C.arg)[oj + i] = P.st_arg[src + i];
      }
    }
    run += all;
    __syncthreads();
  }
}

// every staged warp's words to their final offset: tiles of WC_T staged
// warps (one per thread) claimed through a ticket, a block scan of their
// counts and a decoupled look-back across the tiles (tile_lookback) for the
// tile's offset; each warp then copies its 32 staged warps, coalesced
constexpr int WC_T = 256;

__global__ void __launch_bounds__(WC_T) warp_copy_kernel(const LiveParams P, int64_t nw,
                                                         int64_t n_tiles) {
  __shared__ int64_t s_tile;
  __shared__ uint32_t s_w[WC_T / 32];
  __shared__ uint64_t s_ex;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0)
    s_tile = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(P.ticket), 1ull);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t w = tile * WC_T + threadIdx.x;
  const uint32_t c = w < nw ? P.w_cnt[w] : 0u;
  uint32_t inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t x = lane < WC_T / 32 ? s_w[lane] : 0u;
    uint32_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += u;
    }
    const uint64_t agg = __shfl_sync(0xffffffffu, xi, WC_T / 32 - 1);
    const uint64_t a4[4] = {agg, 0, 0, 0};
    uint64_t e4[4];
    tile_lookback(P.tile_state, tile, a4, e4, lane);
    if (lane < WC_T / 32) s_w[lane] = xi - x;
    if (lane == 0) {
      s_ex = e4[0];
      if (tile == n_tiles - 1) P.C.totals[1] = (int64_t)(e4[0] + agg);
    }
  }
  __syncthreads();
  const uint32_t off = (uint32_t)s_ex + s_w[warp] + inc - c;
  const bool a16 = (P.C.format & PASTE_CF_ARG16) != 0;
  for (int j = 0; j < 32; ++j) {
    const uint32_t cj = __shfl_sync(0xffffffffu, c, j), oj = __shfl_sync(0xffffffffu, off, j);
    if (cj == 0) continue;
    const int64_t src = (tile * WC_T + warp * 32 + j) * 32 * P.M;
    for (uint32_t i = lane; i < cj; i += 32) {
      if (a16)
        static_cast<uint16_t*>(P.C.arg)[oj + i] = reinterpret_cast<const uint16_t*>(P.st_arg)[src + i];
      else
        static_cast<uint32_t*>(P.C.arg)[oj + i] = P.st_arg[src + i];
    }
  }
}

__global__ void __launch_bounds__(LT) live_scatter_kernel(const LiveParams P) {
  __shared__ int64_t s_tile;
  const int64_t n = P.win.n_sessions;
  const paste_compact_desc& C = P.C;
  const bool a16 = (C.format & PASTE_CF_ARG16) != 0;
  const bool entry = (C.format & PASTE_CF_ENTRY16) != 0;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0)
      s_tile = (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(P.ticket), 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= P.n_tiles) break;
    int64_t sj[SCAT_SPT];
    uint32_t cj[SCAT_SPT];
    int c[SCAT_SPT][4];
#pragma unroll
    for (int j = 0; j < SCAT_SPT; ++j) {
      sj[j] = tile * LT * SCAT_SPT + j * LT + threadIdx.x;
      cj[j] = sj[j] < n ? P.st_cnt[sj[j]] : 0u;
      c[j][0] = cj[j] & 31;
      c[j][1] = (cj[j] >> 10) & 0xff;
      c[j][2] = (cj[j] >> 5) & 31;
      c[j][3] = (int)(cj[j] >> 18);
    }
    uint64_t off[SCAT_SPT][4];
    live_offsets<SCAT_SPT>(P, tile, c, off);
#pragma unroll
    for (int j = 0; j < SCAT_SPT; ++j) {
      if (sj[j] >= n || (c[j][0] == 0 && c[j][2] == 0)) continue;
      if ((C.format & PASTE_CF_KEYS) && c[j][1] == 0) continue;
      const int64_t s = sj[j];
      const uint32_t part = c[j][1] > 0 || c[j][2] > 0 ? P.st_part[s] : 0u;
      const uint32_t* sa = P.st_arg + s * P.M;
      for (int q = 0; q < c[j][1]; ++q) {
        const uint32_t w = sa[q];
        if (a16) static_cast<uint16_t*>(C.arg)[off[j][1] + q] = (uint16_t)w;
        else static_cast<uint32_t*>(C.arg)[off[j][1] + q] = w;
      }
      const uint8_t* e = P.plan + (int64_t)P.st_key[s] * P.L.stride;
      if (!entry) {
        const int32_t* pid = reinterpret_cast<const int32_t*>(e + P.L.off_pid);
        const uint8_t* comp = e + P.L.off_comp;
        for (int i = 0; i < c[j][0]; ++i)
          cf_pred(C, off[j][0] + i, pid[i], ((part >> i) & 1u) ? PASTE_C_PARTIAL : comp[i]);
      }
      if (C.format & PASTE_CF_KEYS) continue;  // actions follow from the key
      const uint16_t* act = reinterpret_cast<const uint16_t*>(e + P.L.off_act);
      for (int a = 0; a < c[j][2]; ++a) {
        const uint16_t v = act[a];
        const int slot = v & 0xff;
        const int lv = ((part >> slot) & 1u) ? (v >> 12) & 15 : (v >> 8) & 15;
        C.act[off[j][2] + a] = (uint8_t)(slot | (lv << 5));
      }
    }
  }
}

// Static tiles (tile = CTA + round * grid, every CTA resident, so each
// tile's predecessors are running or done) and the same three-round software
// pipeline as predict_live_kernel: round r+2's inputs and round r+1's older
// ring slots load while round r is keyed, scanned and written.
template <int G>
__global__ void __launch_bounds__(LT) predict_live_compact_pipe_kernel(const LiveParams P) {
  const int64_t n = P.win.n_sessions;
  const int64_t G64 = gridDim.x;
  unsigned long long wide = 0;
  const int64_t t0 = blockIdx.x;
  FrontIn f1, f2;
  Sess<G> y0, y1;
  FrontMid<G> m0, m1;
  front_load(P, t0 * LT + threadIdx.x, f1);
  front_load(P, (t0 + G64) * LT + threadIdx.x, f2);
  front_observe<G>(P, f1, y1, m1);
  for (int64_t tile = t0; tile < P.n_tiles; tile += G64) {
    y0 = y1;
    m0 = m1;
    f1 = f2;
    front_load(P, (tile + 2 * G64) * LT + threadIdx.x, f2);
    front_observe<G>(P, f1, y1, m1);
    front_key<G, true>(P, y0, m0);
    int c[1][4] = {{y0.nm, arg_count(P, y0), y0.n_act, y0.n_err}};
    uint64_t off[1][4];
    live_offsets<1>(P, tile, c, off);
    if (y0.s < n) compact_write<G>(P, y0, off[0], wide);
  }
  if (wide) atomicAdd(reinterpret_cast<unsigned long long*>(P.C.totals + 3), wide);
}

}  // namespace paste

using namespace paste;

static int live_mode();

static int live_gather_depth(const paste_pool_desc* pool, int W) {
  const int g = pool->relation == PASTE_REL_ANCHORED ? pool->k : pool->max_ctx;
  return g < W ? g : W;
}

static int64_t live_keys(const paste_pool_desc* pool, int G) {
  int64_t keys = pool->n_bucket_sigs;
  for (int a = 1; a < G; ++a) keys *= (int64_t)pool->n_bucket_sigs + 1;
  return keys;
}

extern "C" int64_t paste_live_plan_bytes(const paste_pool_desc* pool, int32_t max_candidates,
                                         int32_t window_capacity) {
  if (!pool || !pool->match_table || max_candidates < 1 || max_candidates > 31 ||
      pool->mt_k < max_candidates || window_capacity < 1 || window_capacity > 16)
    return -1;
  const int G = live_gather_depth(pool, window_capacity);
  if (G < 1 || G > 4 || pool->mt_g != G) return -1;
  const PlanLayout L = plan_layout(max_candidates, pool->max_bindings);
  if (L.M > 255) return -1;
  return live_keys(pool, G) * L.stride;
}

extern "C" int paste_build_live_plan(const paste_pool_desc* pool, const paste_admit_desc* admit,
                                     int32_t max_candidates, int32_t window_capacity, void* plan,
                                     void* stream) {
  reset_launches();
  PASTE_REQUIRE(pool && admit && plan, "null argument");
  const int64_t bytes = paste_live_plan_bytes(pool, max_candidates, window_capacity);
  if (bytes < 0) {
    set_error("pool / request shape outside the live-plan envelope (match table, K <= 31, G <= 4)");
    return PASTE_ERR_UNSUPPORTED;
  }
  const int G = live_gather_depth(pool, window_capacity);
  const int64_t keys = live_keys(pool, G);
  const PlanLayout L = plan_layout(max_candidates, pool->max_bindings);
  const int64_t mt_stride = 16 + 32 * (int64_t)pool->mt_k;
  cudaStream_t st = (cudaStream_t)stream;
  PASTE_CUDA_CHECK(cudaMemsetAsync(plan, 0, bytes, st));
  build_live_plan_kernel<<<(unsigned)((keys + 127) / 128), 128, 0, st>>>(
      *pool, *admit, static_cast<const uint8_t*>(pool->match_table), mt_stride, keys, L,
      static_cast<uint8_t*>(plan));
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

extern "C" int64_t paste_live_walk_bytes(int32_t n_bindings, int64_t n_nodes) {
  if (n_bindings < 1 || n_nodes < 1) return -1;
  const int64_t entries = (int64_t)n_bindings * n_nodes;
  return entries > (1ll << 24) ? -1 : 4 * entries;
}

extern "C" int paste_build_live_walk(const paste_pool_desc* pool, int32_t n_bindings,
                                     const paste_tape_node* nodes, int64_t n_nodes, int32_t* walk,
                                     void* stream) {
  reset_launches();
  PASTE_REQUIRE(pool && nodes && walk, "null argument");
  if (paste_live_walk_bytes(n_bindings, n_nodes) < 0) {
    set_error("walk table over 2^24 entries");
    return PASTE_ERR_UNSUPPORTED;
  }
  const int64_t total = (int64_t)n_bindings * n_nodes;
  build_walk_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      *pool, n_bindings, nodes, n_nodes, walk);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

static bool live_ticket() {
  static int t = -1;
  if (t < 0) t = getenv("PASTE_LIVE_TICKET") != nullptr ? 1 : 0;
  return t == 1;
}

// min resident CTAs per SM of the K-slot live kernel, i.e. its register
// cap: 7 -> 72 registers and no spills, the default (per 1M-session step:
// 56 us; 6 -> 80 registers 58 us; 8 -> 64 registers with spills 59 us; 4 ->
// 96 registers 64 us; 10 / 12 -> 48 / 40 registers 77 / 87 us; a pipeline
// one round deeper -- the next round's plan header loaded while this round
// writes -- ran at 60 us with 96 registers and 74 us with spills at 80);
// PASTE_LIVE_MINB = 4 / 5 / 6 / 8 selects another build
static int live_minb() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("PASTE_LIVE_MINB");
    m = e ? atoi(e) : 7;
  }
  return m;
}

template <int G, int SPT>
static void launch_live(const LiveParams& P, bool compact, cudaStream_t st) {
  static int sms = 0;
  static int occ[7] = {0, 0, 0, 0, 0, 0, 0};
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int minb = live_minb();
  const int which = !compact ? (minb == 6 ? 4 : minb == 5 ? 3 : minb == 8 ? 5 : minb == 4 ? 6 : 0)
                             : live_mode() == 1 ? 1 : 2;
  int& o = occ[which];
  if (o == 0) {
    if (which == 0)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, predict_live_kernel<G>, LT, 0);
    else if (which == 3)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, predict_live_kernel<G, 5>, LT, 0);
    else if (which == 4)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, predict_live_kernel<G, 6>, LT, 0);
    else if (which == 5)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, predict_live_kernel<G, 8>, LT, 0);
    else if (which == 6)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, predict_live_kernel<G, 4>, LT, 0);

    else if (which == 1)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, predict_live_compact_kernel<G, SPT>, LT, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, predict_live_compact_pipe_kernel<G>, LT, 0);
    if (o < 1) o = 1;
  }
  const int spt = which == 1 ? SPT : 1;
  const int64_t groups = (P.win.n_sessions + LT * spt - 1) / (LT * spt);
  const int64_t grid = groups < (int64_t)sms * o ? groups : (int64_t)sms * o;
  if (which == 0)
    predict_live_kernel<G><<<(unsigned)grid, LT, 0, st>>>(P);
  else if (which == 3)
    predict_live_kernel<G, 5><<<(unsigned)grid, LT, 0, st>>>(P);
  else if (which == 4)
    predict_live_kernel<G, 6><<<(unsigned)grid, LT, 0, st>>>(P);
  else if (which == 5)
    predict_live_kernel<G, 8><<<(unsigned)grid, LT, 0, st>>>(P);
  else if (which == 6)
    predict_live_kernel<G, 4><<<(unsigned)grid, LT, 0, st>>>(P);

  else if (which == 1)
    predict_live_compact_kernel<G, SPT><<<(unsigned)grid, LT, 0, st>>>(P);
  else
    predict_live_compact_pipe_kernel<G><<<(unsigned)grid, LT, 0, st>>>(P);
}

static int live_spt() {
  static int spt = 0;
  if (spt == 0) {
    const char* e = getenv("PASTE_LIVE_SPT");
    spt = e ? atoi(e) : 2;
    if (spt != 1 && spt != 2 && spt != 4) spt = 2;
  }
  return spt;
}

template <int G>
static void launch_live_g(const LiveParams& P, bool compact, cudaStream_t st) {
  switch (live_spt()) {
    case 1: launch_live<G, 1>(P, compact, st); break;
    case 4: launch_live<G, 4>(P, compact, st); break;
    default: launch_live<G, 2>(P, compact, st); break;
  }
}

static int live_prepare(const paste_pool_desc* pool, paste_windows* w, const paste_admit_desc* adm,
                        const paste_live_plan* plan, int K, LiveParams& P) {
  PASTE_REQUIRE(pool && w && adm && plan && plan->plan, "null argument");
  PASTE_REQUIRE((w->new_tok != nullptr && (w->new_ref || w->new_node)) ||
                    (w->new_tok8 != nullptr &&
                     (w->new_node16 != nullptr || (w->new_node8 != nullptr && w->node_codes != nullptr) ||
                      (w->event_codes != nullptr && !w->new_node16 && !w->new_node8))),
                "the live kernel observes one new event per session");
  PASTE_REQUIRE(!w->stream_end, "stream-mode windows are not live sessions");
  PASTE_REQUIRE(w->capacity >= 1 && w->capacity <= 16, "live plan needs window capacity <= 16");
  PASTE_REQUIRE(plan->max_candidates == K, "plan built for another max_candidates");
  PASTE_REQUIRE(plan->max_bindings == pool->max_bindings, "plan built for another pool");
  const int G = live_gather_depth(pool, w->capacity);
  PASTE_REQUIRE(G >= 1 && G <= 4 && pool->mt_g == G, "plan / window depth mismatch");
  memset(&P, 0, sizeof(P));
  P.pool = *pool;
  P.win = *w;
  P.plan = static_cast<const uint8_t*>(plan->plan);
  P.L = plan_layout(K, pool->max_bindings);
  P.walk = plan->walk;
  P.walk_nodes = plan->walk ? plan->walk_nodes : 0;
  P.admit = adm->enabled;
  P.S = pool->n_bucket_sigs;
  return PASTE_OK;
}

template <typename F>
static void by_depth(int G, F f) {
  switch (G) {
    case 1: f(std::integral_constant<int, 1>()); break;
    case 2: f(std::integral_constant<int, 2>()); break;
    case 3: f(std::integral_constant<int, 3>()); break;
    default: f(std::integral_constant<int, 4>()); break;
  }
}

extern "C" int paste_predict_live(const paste_pool_desc* pool, paste_windows* windows,
                                  const paste_admit_desc* admit, const paste_live_plan* plan,
                                  paste_predict_out* out, void* stream) {
  reset_launches();
  PASTE_REQUIRE(out != nullptr, "null output");
  PASTE_REQUIRE(out->max_bindings >= pool->max_bindings, "max_bindings below pool maximum");
  LiveParams P;
  const int rc = live_prepare(pool, windows, admit, plan, out->max_candidates, P);
  if (rc != PASTE_OK) return rc;
  P.out = *out;
  P.fast8 = out->max_candidates == 8 && out->slot_major &&
            windows->n_sessions * 8 * (int64_t)out->max_bindings < (1ll << 31);
  if (windows->n_sessions == 0) return PASTE_OK;
  const int G = live_gather_depth(pool, windows->capacity);
  cudaStream_t st = (cudaStream_t)stream;
  by_depth(G, [&](auto g) { launch_live_g<decltype(g)::value>(P, false, st); });
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

static int64_t live_state_bytes(int64_t n) {
  const int64_t tiles = (n + LT - 1) / LT;  // the most tiles any mode uses
  return (8 * (LB_STRIDE * tiles + LB_STRIDE) + 255) / 256 * 256;
}

extern "C" int64_t paste_predict_live_compact_scratch_bytes(int64_t n_sessions,
                                                            int32_t max_candidates,
                                                            int32_t max_bindings) {
  const int64_t M = (int64_t)max_candidates * (max_bindings > 0 ? max_bindings : 1);
  const int64_t n = n_sessions, n32 = (n + 31) / 32 * 32;  // warp staging slots: whole warps
  return live_state_bytes(n) + 3 * ((4 * n + 255) / 256 * 256) + (4 * n32 * M + 255) / 256 * 256;
}

// 0 two-pass (default; the key-stream form runs the warp-staged kernels),
// 1 ticket tiles, 2 pipelined static tiles, 3 two-pass with the tile
// look-back scatter for the key-stream form too
static int live_mode_impl() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("PASTE_LIVE_MODE");
    m = !e ? 0 : !strcmp(e, "ticket") ? 1 : !strcmp(e, "pipe") ? 2 : !strcmp(e, "scatter") ? 3 : 0;
    if (live_ticket()) m = 1;
  }
  return m;
}

static bool live_coop() {  // PASTE_LIVE_COOP=0: step + look-back copy as two launches
  static int c = -1;
  if (c < 0) {
    const char* e = getenv("PASTE_LIVE_COOP");
    c = e && !strcmp(e, "0") ? 0 : 1;
  }
  return c == 1;
}

template <int G>
static void launch_keys(const LiveParams& P, cudaStream_t st) {
  if (live_coop()) {
    // register cap: 6 CTAs/SM -> 80 registers, no spills (38.9 us per 1M
    // sessions queued); PASTE_LIVE_KEYS_MINB=7 -> 72 registers, 44 B spilled
    // (40.6 us)
    static int minb = 0;
    if (minb == 0) {
      const char* e = getenv("PASTE_LIVE_KEYS_MINB");
      minb = e && atoi(e) == 7 ? 7 : 6;
    }
    const void* fn = minb == 6 ? (const void*)predict_live_keys_coop_kernel<G, 6>
                               : (const void*)predict_live_keys_coop_kernel<G, 7>;
    static int sms = 0, oc = 0;
    if (sms == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, fn, LT, 0);
      if (oc < 1) oc = 1;
    }
    const int64_t g1 = (P.win.n_sessions + LT - 1) / LT;
    const unsigned grid = (unsigned)(g1 < (int64_t)sms * oc ? g1 : (int64_t)sms * oc);
    LiveParams Q = P;
    void* args[] = {&Q};
    cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(LT), args, 0, st);
    return;
  }
  static int sms = 0, o1 = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, predict_live_keys_kernel<G, 7>, LT, 0);
    if (o1 < 1) o1 = 1;
  }
  const int64_t n = P.win.n_sessions;
  const int64_t nw = (n + 31) / 32;
  const int64_t g1 = (n + LT - 1) / LT;
  predict_live_keys_kernel<G, 7><<<(unsigned)(g1 < (int64_t)sms * o1 ? g1 : (int64_t)sms * o1), LT,
                                   0, st>>>(P);
  warp_copy_kernel<<<(unsigned)P.n_tiles, WC_T, 0, st>>>(P, nw, P.n_tiles);
}

static int live_mode() { return live_mode_impl(); }

template <int G>
static void launch_two_pass(const LiveParams& P, cudaStream_t st) {
  static int sms = 0, o1 = 0, o2 = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, predict_live_stage_kernel<G>, LT, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, live_scatter_kernel, LT, 0);
    if (o1 < 1) o1 = 1;
    if (o2 < 1) o2 = 1;
  }
  const int64_t n = P.win.n_sessions;
  const int64_t g1 = (n + LT - 1) / LT;
  predict_live_stage_kernel<G><<<(unsigned)(g1 < (int64_t)sms * o1 ? g1 : (int64_t)sms * o1), LT,
                                 0, st>>>(P);
  const int64_t g2 = P.n_tiles < (int64_t)sms * o2 ? P.n_tiles : (int64_t)sms * o2;
  live_scatter_kernel<<<(unsigned)g2, LT, 0, st>>>(P);
}

extern "C" int paste_predict_live_compact(const paste_pool_desc* pool, paste_windows* windows,
                                          const paste_admit_desc* admit,
                                          const paste_live_plan* plan, int32_t max_bindings,
                                          paste_compact_desc* c, void* scratch,
                                          int64_t scratch_bytes, void* stream) {
  reset_launches();
  PASTE_REQUIRE(c != nullptr && scratch != nullptr, "null argument");
  PASTE_REQUIRE(max_bindings >= pool->max_bindings, "max_bindings below pool maximum");
  LiveParams P;
  const int rc = live_prepare(pool, windows, admit, plan, plan->max_candidates, P);
  if (rc != PASTE_OK) return rc;
  const int K = plan->max_candidates;
  if (((c->format & PASTE_CF_HDR8) && K > 15) ||
      ((c->format & PASTE_CF_PRED8) && pool->n_patterns > 64) || pool->n_patterns > (1 << 14) ||
      ((c->format & PASTE_CF_ENTRY16) &&
       live_keys(pool, live_gather_depth(pool, windows->capacity)) >= 0xffff) ||
      ((c->format & PASTE_CF_KEYS) && !(c->format & PASTE_CF_ENTRY16)) ||
      ((c->format & PASTE_CF_UNIQ) && !(c->format & PASTE_CF_KEYS)) ||
      ((c->format & PASTE_CF_KEY8) && !(c->format & PASTE_CF_KEYS))) {
    set_error("stream format outside the live plan's envelope");
    return PASTE_ERR_UNSUPPORTED;
  }
  const int64_t n = windows->n_sessions;
  const int64_t need = paste_predict_live_compact_scratch_bytes(n, K, max_bindings);
  PASTE_REQUIRE(scratch_bytes >= need, "scratch too small (%lld bytes)", (long long)need);
  P.C = *c;
  const int mode = live_mode();
  const int spt = mode == 1 ? live_spt() : (mode == 0 || mode == 3) ? SCAT_SPT : 1;
  P.n_tiles = (n + LT * spt - 1) / (LT * spt);
  P.ticket = static_cast<uint64_t*>(scratch);
  P.tile_state = static_cast<uint64_t*>(scratch) + LB_STRIDE;
  uint8_t* stg = static_cast<uint8_t*>(scratch) + live_state_bytes(n);
  const int64_t a4 = (4 * n + 255) / 256 * 256;
  P.st_key = reinterpret_cast<int32_t*>(stg);
  P.st_cnt = reinterpret_cast<uint32_t*>(stg + a4);
  P.st_part = reinterpret_cast<uint32_t*>(stg + 2 * a4);
  P.st_arg = reinterpret_cast<uint32_t*>(stg + 3 * a4);
  P.M = K * (max_bindings > 0 ? max_bindings : 1);
  P.w_cnt = reinterpret_cast<uint32_t*>(stg);        // key-stream form: [n / 32]
  cudaStream_t st = (cudaStream_t)stream;
  const bool keys_form = mode == 0 && (c->format & PASTE_CF_KEYS) &&
                         ((n + 31) / 32) * 32 * (int64_t)P.M < (1ll << 32);
  if (keys_form) P.n_tiles = ((n + 31) / 32 + WC_T - 1) / WC_T;  // warp_copy_kernel tiles
  if (!keys_form)
    PASTE_CUDA_CHECK(cudaMemsetAsync(scratch, 0, 8 * (LB_STRIDE * P.n_tiles + LB_STRIDE), st));
  PASTE_CUDA_CHECK(cudaMemsetAsync(c->totals, 0, 5 * sizeof(int64_t), st));
  if (n == 0) return PASTE_OK;
  const int G = live_gather_depth(pool, windows->capacity);
  if (keys_form) {
    by_depth(G, [&](auto g) { launch_keys<decltype(g)::value>(P, st); });
    count_launch(live_coop() ? 1 : 2);
  } else if (mode == 0 || mode == 3) {
    by_depth(G, [&](auto g) { launch_two_pass<decltype(g)::value>(P, st); });
    count_launch(2);
  } else {
    by_depth(G, [&](auto g) { launch_live_g<decltype(g)::value>(P, true, st); });
    count_launch();
  }
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
