// K4 predict_topk_admit: batched Predictor.predict + admit for live sessions.
//
// Reference semantics (paths relative to /root/reference/pkg/src/spectool):
//   Predictor.predict        prediction.py:76-118
//   match_at                 mining.py:119-156
//   evaluate / _resolve      mappings.py:143-223
//   admit / _beats           policy.py:207-244
//
// Design (one thread per session):
//   * the window is a ring of W (token, event) slots; only the last G tool
//     events matter (G = k for anchored subsequence, max context length for
//     contiguous suffix), so the thread gathers those from the ring and never
//     touches the rest of the window;
//   * the pool is bucketed by the last context signature and each bucket is
//     pre-sorted on the host by the static rank (-p, pattern_id, pool index):
//     the first K matches in bucket order ARE the reference's sorted, truncated
//     list, so no per-session sort is needed;
//   * mapping evaluation walks the payload tapes of the matched events only;
//   * the admit epilogue (policy level, utility = p * benefit, per-tool
//     arbitration) runs on the thread's K candidates in registers/local memory.
#include <stdlib.h>

#include "common.cuh"

namespace paste {

constexpr int GMAX = 16;  // gathered tool events (max k / context length)

struct PredictParams {
  paste_pool_desc pool;
  paste_windows win;
  paste_admit_desc adm;
  paste_predict_out out;
};

// Resolve one binding.  `gtok`/`gslot` are the gathered (oldest..newest) window
// positions, `mpos[j]` the gathered position of context element j.
__device__ __forceinline__ int64_t resolve_binding(const PredictParams& P, const paste_binding& bd,
                                                   const int32_t* gtok, const int32_t* gslot,
                                                   const int32_t* mpos, int m, int64_t sess) {
  const int src = mpos[bd.ctx_pos];
  // plain load: the slot may have been written by this thread's observe step
  const int32_t ev = P.win.evt[ring_at(P.win, sess, gslot[src])];
  const paste_event_ref ref = P.win.refs[ev];
  const int64_t base = ref.node_base;
  const int32_t* steps = P.pool.steps;
  int64_t cur = 0;
  if (bd.kind == PASTE_X_FALLBACK) {
    // index = start + #FAIL(fail_tool) after the source (mappings.py:167-194)
    if (bd.start_index < 0) return -1;
    int fails = 0;
    for (int q = src + 1; q < m; ++q) {
      const int32_t t = gtok[q];
      fails += ((t >> 1) == bd.fail_tool) && ((t & 1) == 0);
    }
    for (int s = 0; s < bd.step_cnt && cur >= 0; ++s)
      cur = step_child(P.win.nodes, base, cur, steps[2 * (bd.step_off + s)],
                       steps[2 * (bd.step_off + s) + 1]);
    if (cur < 0) return -1;
    cur = step_child(P.win.nodes, base, cur, 1, bd.start_index + fails);
    for (int s = 0; s < bd.suf_cnt && cur >= 0; ++s)
      cur = step_child(P.win.nodes, base, cur, steps[2 * (bd.suf_off + s)],
                       steps[2 * (bd.suf_off + s) + 1]);
  } else {
    for (int s = 0; s < bd.step_cnt && cur >= 0; ++s)
      cur = step_child(P.win.nodes, base, cur, steps[2 * (bd.step_off + s)],
                       steps[2 * (bd.step_off + s) + 1]);
    if (cur >= 0 && bd.kind == PASTE_X_FORMAT) {
      // _leaf_str: only str / number leaves fill the hole (mappings.py:197-204)
      const int t = load_node(P.win.nodes, base + cur).type();
      if (t != PASTE_T_STR && t != PASTE_T_INT && t != PASTE_T_FLOAT) cur = -1;
    }
  }
  if (cur < 0) return -1;
  return ((int64_t)ev << 32) | (int64_t)cur;
}

__global__ void __launch_bounds__(256) predict_kernel(const PredictParams P) {
  const int64_t sess = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sess >= P.win.n_sessions) return;
  const int W = P.win.capacity;
  int64_t cnt = P.win.count[sess];

  // observe (PredictionWindow.observe: deque append with maxlen W)
  if (P.win.new_tok != nullptr) {
    const int slot = (int)(cnt % W);
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
    P.win.tok[ring_at(P.win, sess, slot)] = P.win.new_tok[sess];
    P.win.evt[ring_at(P.win, sess, slot)] = (int32_t)ev;
    ++cnt;
    P.win.count[sess] = cnt;
  }
  const int len = (int)(cnt < W ? cnt : W);
  const paste_pool_desc& pool = P.pool;
  // anchored: the embedding may skip events, so all of the last k count
  const int G = min(pool.relation == PASTE_REL_ANCHORED ? pool.k : pool.max_ctx, W);

  // gather the newest G tool events, stored oldest..newest
  int32_t gtok[GMAX], gslot[GMAX];
  int m = 0;
  {
    int32_t rt[GMAX], rs[GMAX];
    for (int i = 0; i < len && m < G; ++i) {
      const int slot = (int)((cnt - 1 - i) % W);
      const int32_t t = P.win.tok[ring_at(P.win, sess, slot)];
      if (t >= 0) {
        rt[m] = t;
        rs[m] = slot;
        ++m;
      }
    }
    for (int i = 0; i < m; ++i) {
      gtok[i] = rt[m - 1 - i];
      gslot[i] = rs[m - 1 - i];
    }
  }

  const int K = P.out.max_candidates;
  int n_pred = 0, n_err = 0;
  // candidate state kept for the admit epilogue
  int32_t cpat[GMAX * 2];
  uint8_t ccomp[GMAX * 2];
  const int KC = K < GMAX * 2 ? K : GMAX * 2;  // epilogue handles <=32 in registers

  if (m > 0 && gtok[m - 1] < pool.n_bucket_sigs) {
    const int a = gtok[m - 1];
    const int b0 = __ldg(pool.bucket_off + a), b1 = __ldg(pool.bucket_off + a + 1);
    const bool scan_all = __ldg(pool.bucket_scan_all + a) != 0;
    for (int bi = b0; bi < b1; ++bi) {
      const int pid = __ldg(pool.bucket_pat + bi);
      const paste_pattern pt = pool.patterns[pid];
      const int n = pt.ctx_len;
      int32_t mpos[GMAX];
      bool ok;
      if (pool.relation == PASTE_REL_ANCHORED) {
        // rightmost embedding within the last k events (mining.py:142-155)
        if (n > GMAX) continue;
        mpos[n - 1] = m - 1;
        int j = n - 2, pos = m - 2;
        while (j >= 0 && pos >= 0) {
          if (gtok[pos] == __ldg(pool.ctx_sig + pt.ctx_off + j)) mpos[j--] = pos;
          --pos;
        }
        ok = j < 0;
      } else {
        // exact slice ending at the anchor (mining.py:133-140)
        ok = n <= m;
        for (int i = 0; ok && i < n - 1; ++i)
          ok = gtok[m - n + i] == __ldg(pool.ctx_sig + pt.ctx_off + i);
        if (ok)
          for (int i = 0; i < n; ++i) mpos[i] = m - n + i;
      }
      if (!ok) continue;
      if (pt.flags & PASTE_PF_STRUCT_ERR) {  // MappingStructureError: tallied, skipped
        ++n_err;
        continue;
      }
      if (n_pred >= K) {
        if (!scan_all) break;
        continue;
      }
      const int64_t slot = out_at(P.out, P.win.n_sessions, sess, n_pred);
      uint8_t comp;
      if (!(pt.flags & PASTE_PF_HAS_MAPPING)) {
        comp = PASTE_C_TOOL_ONLY;
      } else {
        comp = PASTE_C_FULL;
        for (int bi2 = 0; bi2 < pt.n_bind; ++bi2) {
          const paste_binding bd = pool.bindings[pt.bind_off + bi2];
          const int64_t r = resolve_binding(P, bd, gtok, gslot, mpos, m, sess);
          if (r < 0) comp = PASTE_C_PARTIAL;
          P.out.pred_arg[arg_at(P.out, P.win.n_sessions, sess, n_pred, bi2)] = r;
        }
      }
      P.out.pred_pat[slot] = pid;
      P.out.pred_comp[slot] = comp;
      if (n_pred < KC) {
        cpat[n_pred] = pid;
        ccomp[n_pred] = comp;
      }
      ++n_pred;
      if (n_pred >= K && !scan_all) break;
    }
  }
  P.out.n_pred[sess] = n_pred;
  P.out.struct_err[sess] = n_err;

  if (!P.adm.enabled) return;
  // admit (policy.py:207-236): first-appearance order, one action per tool
  int n_act = 0;
  int32_t atool[GMAX * 2];
  int16_t apred[GMAX * 2];
  double autil[GMAX * 2], ap[GMAX * 2];
  uint8_t alevel[GMAX * 2];
  for (int i = 0; i < n_pred && i < KC; ++i) {
    const paste_pattern pt = pool.patterns[cpat[i]];
    const int tool = pt.target_tool;
    const bool allow = tool < P.adm.n_tools ? __ldg(P.adm.allow + tool) != 0 : false;
    if (!allow) continue;
    const int implied = ccomp[i] == PASTE_C_FULL ? 3 : 1;
    const int cap = __ldg(P.adm.max_level + tool);
    const int level = cap < implied ? cap : implied;
    const double util = __dmul_rn(pt.p, __ldg(P.adm.benefit + tool));
    int j = 0;
    while (j < n_act && atool[j] != tool) ++j;
    if (j == n_act) {
      atool[j] = tool;
      apred[j] = (int16_t)i;
      autil[j] = util;
      ap[j] = pt.p;
      alevel[j] = (uint8_t)level;
      ++n_act;
    } else {
      // _beats: (utility, p, -created_at) lexicographic; created_at is shared
      const bool beats = (util != autil[j]) ? (util > autil[j]) : (pt.p > ap[j]);
      if (beats) {
        apred[j] = (int16_t)i;
        autil[j] = util;
        ap[j] = pt.p;
        alevel[j] = (uint8_t)level;
      }
    }
  }
  P.out.n_act[sess] = n_act;
  for (int j = 0; j < n_act; ++j) {
    const int64_t o = out_at(P.out, P.win.n_sessions, sess, j);
    P.out.act_pred[o] = apred[j];
    P.out.act_level[o] = alevel[j];
    P.out.act_util[o] = autil[j];
  }
}

}  // namespace paste

extern "C" int paste_predict_batch(const paste_pool_desc* pool, paste_windows* windows,
                                   const paste_admit_desc* admit, paste_predict_out* out,
                                   void* stream) {
  using namespace paste;
  reset_launches();
  PASTE_REQUIRE(pool && windows && admit && out, "null descriptor");
  PASTE_REQUIRE(windows->capacity >= 1, "window capacity must be >= 1");
  PASTE_REQUIRE(out->max_candidates >= 1, "max_candidates must be >= 1");
  PASTE_REQUIRE(out->max_bindings >= pool->max_bindings, "max_bindings below pool maximum");
  PASTE_REQUIRE(pool->k >= 1, "k must be >= 1");
  PASTE_REQUIRE(!(windows->stream_end && windows->new_tok), "stream-mode windows cannot observe");
  PASTE_REQUIRE(!windows->new_tok8 && !windows->new_node16 && !windows->new_node8,
                "the narrow observe form needs the live-plan kernel (paste_predict_live)");
  {
    const int g = pool->relation == PASTE_REL_ANCHORED ? pool->k : pool->max_ctx;
    if ((g < windows->capacity ? g : windows->capacity) > GMAX) {
      set_error("min(%s, window capacity) = %d exceeds the device envelope (%d)",
                pool->relation == PASTE_REL_ANCHORED ? "k" : "max context",
                g < windows->capacity ? g : windows->capacity, GMAX);
      return PASTE_ERR_UNSUPPORTED;
    }
  }
  if (admit->enabled && out->max_candidates > GMAX * 2) {
    set_error("admit epilogue supports at most %d candidates per session", GMAX * 2);
    return PASTE_ERR_UNSUPPORTED;
  }
  if (windows->n_sessions == 0) return PASTE_OK;
  {
    const int g = pool->relation == PASTE_REL_ANCHORED ? pool->k : pool->max_ctx;
    const int G = g < windows->capacity ? g : windows->capacity;
    // PASTE_FORCE_GENERIC=1 pins the generic kernel (A/B parity tests)
    static const bool force_generic = getenv("PASTE_FORCE_GENERIC") != nullptr;
    if (!force_generic &&
        predict_fast_dispatch(pool, windows, admit, out, G, (cudaStream_t)stream)) {
      count_launch();
      PASTE_CUDA_CHECK(cudaGetLastError());
      return PASTE_OK;
    }
  }
  PredictParams P{*pool, *windows, *admit, *out};
  const int threads = 256;
  const int64_t blocks = (windows->n_sessions + threads - 1) / threads;
  predict_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(P);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

// ---------------------------------------------------------------------------
// Standalone admit over prediction lists (policy.py:207-244).  One thread per
// list; the list's actions are built in place in its own output slots.
// ---------------------------------------------------------------------------
namespace paste {

__global__ void admit_lists_kernel(const paste_admit_desc adm, const paste_admit_lists_desc L) {
  const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= L.n_lists) return;
  const int64_t b0 = L.list_off[li], b1 = L.list_off[li + 1];
  int n_act = 0;
  for (int64_t i = b0; i < b1; ++i) {
    const int tool = L.tool[i];
    if (tool < 0 || tool >= adm.n_tools || !adm.allow[tool]) continue;
    const int implied = L.full[i] ? 3 : 1;
    const int cap = adm.max_level[tool];
    const int level = cap < implied ? cap : implied;
    const double util = __dmul_rn(L.p[i], L.benefit[i]);
    int j = 0;
    while (j < n_act && L.tool[b0 + L.act_pred[b0 + j]] != tool) ++j;
    if (j == n_act) {
      L.act_pred[b0 + j] = (int32_t)(i - b0);
      L.act_level[b0 + j] = (uint8_t)level;
      L.act_util[b0 + j] = util;
      ++n_act;
      continue;
    }
    // _beats: lexicographic (utility, p, -created_at), strict
    const int64_t inc = b0 + L.act_pred[b0 + j];
    const double iu = L.act_util[b0 + j];
    bool beats;
    if (util != iu) beats = util > iu;
    else if (L.p[i] != L.p[inc]) beats = L.p[i] > L.p[inc];
    else beats = -L.created_at[i] > -L.created_at[inc];
    if (beats) {
      L.act_pred[b0 + j] = (int32_t)(i - b0);
      L.act_level[b0 + j] = (uint8_t)level;
      L.act_util[b0 + j] = util;
    }
  }
  L.n_act[li] = n_act;
}

}  // namespace paste

extern "C" int paste_admit_lists(const paste_admit_desc* policy, paste_admit_lists_desc* lists,
                                 void* stream) {
  using namespace paste;
  reset_launches();
  PASTE_REQUIRE(policy && lists, "null descriptor");
  if (lists->n_lists == 0) return PASTE_OK;
  const int threads = 128;
  const int64_t blocks = (lists->n_lists + threads - 1) / threads;
  admit_lists_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(*policy, *lists);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
