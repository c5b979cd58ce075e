/*
 * paste_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's hot-path algorithms
 * (spectool, /root/reference/pkg/src/spectool), operating on the same packed
 * inputs as libpaste (include/paste.h) so its outputs can be compared with
 * the CUDA kernels record for record.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it; the
 * product path never does.
 *
 * It deliberately follows the reference's control flow rather than the
 * device's shortcuts: predict scans the whole pool in pool order, collects
 * every match and sorts by (-p, pattern_id) with a stable sort
 * (prediction.py:88-117) instead of using pre-ranked buckets; admit keeps
 * incumbents in a map keyed by tool (policy.py:207-244).
 *
 * Pinning: tests/test_oracle_golden.py checks this oracle (through the host
 * packing/decoding of paper_2603_18897_b200) against golden vectors produced
 * by running the reference itself (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "paste.h"

/* ring / output addressing (session-major or slot-major, include/paste.h) */
static int64_t ring_idx(const paste_windows* w, int64_t s, int slot) {
  if (w->stream_end) return w->stream_end[s] - w->count[s] + slot; /* stream mode: count <= W */
  return w->slot_major ? (int64_t)slot * w->n_sessions + s : s * w->capacity + slot;
}
static int64_t out_idx(const paste_predict_out* o, int64_t n, int64_t s, int i) {
  return o->slot_major ? (int64_t)i * n + s : s * o->max_candidates + i;
}
static int64_t arg_idx(const paste_predict_out* o, int64_t n, int64_t s, int i, int b) {
  return o->slot_major ? ((int64_t)i * o->max_bindings + b) * n + s
                       : (s * o->max_candidates + i) * o->max_bindings + b;
}

typedef struct {
  const paste_tape_node* nodes;
  const paste_event_ref* refs;
} tapes_t;


static uint32_t node_size(const paste_tape_node* n) {
  return n->type >= PASTE_T_LIST ? n->b : 1u;
}

/* _walk (mappings.py:143-153) over one step; returns child or -1 */
static int64_t walk_step(const tapes_t* T, int64_t base, int64_t cur, int32_t kind, int32_t value) {
  const paste_tape_node* nd = &T->nodes[base + cur];
  int64_t child = cur + 1;
  uint32_t c;
  if (kind == 0) { /* str step: node must be a dict holding the key */
    if (nd->type != PASTE_T_DICT) return -1;
    for (c = 0; c < nd->a; ++c) {
      if (T->nodes[base + child].key == value) return child;
      child += node_size(&T->nodes[base + child]);
    }
    return -1;
  }
  /* int step: node must be a list and 0 <= step < len */
  if (nd->type != PASTE_T_LIST || value < 0 || (uint32_t)value >= nd->a) return -1;
  for (c = 0; c < (uint32_t)value; ++c) child += node_size(&T->nodes[base + child]);
  return child;
}

static int64_t walk_path(const tapes_t* T, int64_t base, int64_t cur, const int32_t* steps,
                         int32_t off, int32_t cnt) {
  int32_t s;
  for (s = 0; s < cnt && cur >= 0; ++s)
    cur = walk_step(T, base, cur, steps[2 * (off + s)], steps[2 * (off + s) + 1]);
  return cur;
}

typedef struct {
  double p;
  const char* pid;
  int32_t pat;
  int32_t pool_order;
  uint8_t comp;
  int64_t args[64];
} cand_t;

/* stable insertion sort by (-p, pattern_id) -- prediction.py:115 */
static int cand_before(const cand_t* a, const cand_t* b) {
  if (a->p != b->p) return a->p > b->p;
  return strncmp(a->pid, b->pid, 16) < 0;
}

/* One session: Predictor.predict (prediction.py:76-118) + admit (policy.py:207-244). */
static void predict_one(const paste_pool_desc* pool, const char* pids, const paste_windows* win,
                        const paste_admit_desc* adm, paste_predict_out* out, int64_t s,
                        cand_t* cands, int32_t* stream_tok, int32_t* stream_slot) {
  const int W = win->capacity;
  const int K = out->max_candidates;
  const int64_t N = win->n_sessions;
  int64_t cnt = win->count[s];
  int len, i, n_stream = 0, n_cand = 0, n_err = 0, p;
  tapes_t T = {win->nodes, win->refs};

  if (win->new_tok) { /* PredictionWindow.observe */
    const int64_t ev = win->new_evt_base + s;
    win->refs[ev].node_base = win->new_ref[s].node_base;
    win->refs[ev].byte_base = win->new_ref[s].byte_base + win->new_byte_base;
    win->tok[ring_idx(win, s, (int)(cnt % W))] = win->new_tok[s];
    win->evt[ring_idx(win, s, (int)(cnt % W))] = (int32_t)ev;
    win->count[s] = ++cnt;
  }
  len = (int)(cnt < W ? cnt : W);
  /* window.tool_events(): oldest..newest */
  for (i = 0; i < len; ++i) {
    int slot = (int)((cnt - len + i) % W);
    if (win->tok[ring_idx(win, s, slot)] >= 0) {
      stream_tok[n_stream] = win->tok[ring_idx(win, s, slot)];
      stream_slot[n_stream] = slot;
      ++n_stream;
    }
  }
  out->n_pred[s] = 0;
  out->struct_err[s] = 0;
  if (adm->enabled) out->n_act[s] = 0;
  if (n_stream == 0) return;
  {
    const int anchor = n_stream - 1;
    for (p = 0; p < pool->n_patterns; ++p) {
      const paste_pattern* pt = &pool->patterns[p];
      const int32_t* ctx = pool->ctx_sig + pt->ctx_off;
      const int n = pt->ctx_len;
      int mpos[64], first_pos, ok = 1, b;
      uint8_t comp;
      if (n == 0 || n > 64 || ctx[n - 1] != stream_tok[anchor]) continue; /* bucket */
      /* match_at (mining.py:119-156) */
      if (pool->relation == PASTE_REL_SUFFIX) {
        int start = anchor - n + 1;
        if (start < 0) continue;
        for (i = 0; i < n; ++i)
          if (stream_tok[start + i] != ctx[i]) { ok = 0; break; }
        if (!ok) continue;
        for (i = 0; i < n; ++i) mpos[i] = start + i;
        first_pos = start;
      } else {
        int lo = anchor - pool->k + 1, j = n - 2, pos = anchor - 1;
        if (lo < 0) lo = 0;
        mpos[n - 1] = anchor;
        while (j >= 0 && pos >= lo) {
          if (stream_tok[pos] == ctx[j]) mpos[j--] = pos;
          --pos;
        }
        if (j >= 0) continue;
        first_pos = mpos[0];
      }
      /* evaluate (mappings.py:207-223); ctx_pos out of range raises
       * MappingStructureError, which predict tallies and skips. */
      comp = PASTE_C_TOOL_ONLY;
      if (pt->flags & PASTE_PF_HAS_MAPPING) {
        int bad = 0;
        for (b = 0; b < pt->n_bind; ++b) {
          int cp = pool->bindings[pt->bind_off + b].ctx_pos;
          if (cp < 0 || cp >= n) bad = 1;
        }
        if (bad) { ++n_err; continue; }
        comp = PASTE_C_FULL;
        for (b = 0; b < pt->n_bind; ++b) {
          const paste_binding* bd = &pool->bindings[pt->bind_off + b];
          const int src = mpos[bd->ctx_pos];
          const int32_t ev = win->evt[ring_idx(win, s, stream_slot[src])];
          const int64_t base = T.refs[ev].node_base;
          int64_t cur;
          if (bd->kind == PASTE_X_FALLBACK) {
            /* _failures_after over history = stream[first_pos..anchor] */
            int fails = 0, q;
            for (q = first_pos; q <= anchor; ++q)
              if (q > src && (stream_tok[q] >> 1) == bd->fail_tool && !(stream_tok[q] & 1)) ++fails;
            cur = walk_path(&T, base, 0, pool->steps, bd->step_off, bd->step_cnt);
            if (cur >= 0) cur = bd->start_index < 0 ? -1 : walk_step(&T, base, cur, 1, bd->start_index + fails);
            if (cur >= 0) cur = walk_path(&T, base, cur, pool->steps, bd->suf_off, bd->suf_cnt);
          } else {
            cur = walk_path(&T, base, 0, pool->steps, bd->step_off, bd->step_cnt);
            if (cur >= 0 && bd->kind == PASTE_X_FORMAT) {
              int t = T.nodes[base + cur].type; /* _leaf_str: str or number */
              if (t != PASTE_T_STR && t != PASTE_T_INT && t != PASTE_T_FLOAT) cur = -1;
            }
          }
          if (cur < 0) comp = PASTE_C_PARTIAL;
          cands[n_cand].args[b] = cur < 0 ? -1 : (((int64_t)ev << 32) | cur);
        }
      }
      cands[n_cand].p = pt->p;
      cands[n_cand].pid = pids + 16 * (int64_t)p;
      cands[n_cand].pat = p;
      cands[n_cand].pool_order = p;
      cands[n_cand].comp = comp;
      /* stable insertion */
      {
        cand_t tmp = cands[n_cand];
        int at = n_cand;
        while (at > 0 && cand_before(&tmp, &cands[at - 1])) {
          cands[at] = cands[at - 1];
          --at;
        }
        cands[at] = tmp;
      }
      ++n_cand;
    }
  }
  out->struct_err[s] = n_err;
  if (n_cand > K) n_cand = K; /* predictions[:max_candidates] */
  out->n_pred[s] = n_cand;
  for (i = 0; i < n_cand; ++i) {
    const int64_t slot = out_idx(out, N, s, i);
    const paste_pattern* pt = &pool->patterns[cands[i].pat];
    int b;
    out->pred_pat[slot] = cands[i].pat;
    out->pred_comp[slot] = cands[i].comp;
    if (cands[i].comp != PASTE_C_TOOL_ONLY)
      for (b = 0; b < pt->n_bind; ++b) out->pred_arg[arg_idx(out, N, s, i, b)] = cands[i].args[b];
  }
  if (!adm->enabled) return;
  {
    /* admit: best[tool] with first-appearance order */
    int n_act = 0, j;
    for (i = 0; i < n_cand; ++i) {
      const paste_pattern* pt = &pool->patterns[cands[i].pat];
      const int tool = pt->target_tool;
      int implied, cap, level;
      double util;
      if (tool >= adm->n_tools || !adm->allow[tool]) continue;
      implied = cands[i].comp == PASTE_C_FULL ? 3 : 1;
      cap = adm->max_level[tool];
      level = cap < implied ? cap : implied;
      util = pt->p * adm->benefit[tool];
      for (j = 0; j < n_act; ++j)
        if (pool->patterns[cands[out->act_pred[out_idx(out, N, s, j)]].pat].target_tool == tool) break;
      if (j == n_act) {
        out->act_pred[out_idx(out, N, s, j)] = (int16_t)i;
        out->act_level[out_idx(out, N, s, j)] = (uint8_t)level;
        out->act_util[out_idx(out, N, s, j)] = util;
        ++n_act;
      } else {
        const double iu = out->act_util[out_idx(out, N, s, j)];
        const double ip = pool->patterns[cands[out->act_pred[out_idx(out, N, s, j)]].pat].p;
        int beats = (util != iu) ? (util > iu) : (pt->p > ip);
        if (beats) {
          out->act_pred[out_idx(out, N, s, j)] = (int16_t)i;
          out->act_level[out_idx(out, N, s, j)] = (uint8_t)level;
          out->act_util[out_idx(out, N, s, j)] = util;
        }
      }
    }
    out->n_act[s] = n_act;
  }
}

/* Batched oracle predict.  All pointers are HOST pointers.  `pids` holds the
 * pattern ids as 16-byte NUL-padded strings. */
int oracle_predict_batch(const paste_pool_desc* pool, const char* pids, paste_windows* win,
                         const paste_admit_desc* adm, paste_predict_out* out, int n_threads) {
  int64_t s;
  if (pool->max_bindings > 64) return PASTE_ERR_UNSUPPORTED;
#pragma omp parallel num_threads(n_threads > 0 ? n_threads : 1)
  {
    cand_t* cands = (cand_t*)malloc(sizeof(cand_t) * (size_t)(pool->n_patterns + 1));
    int32_t* st = (int32_t*)malloc(sizeof(int32_t) * (size_t)win->capacity * 2);
#pragma omp for schedule(static)
    for (s = 0; s < win->n_sessions; ++s)
      predict_one(pool, pids, win, adm, out, s, cands, st, st + win->capacity);
    free(cands);
    free(st);
  }
  return PASTE_OK;
}

/* ------------------------------------------------------------------------ */
/* Mining counts (mine(), mining.py:248-292), restated per the reference:    */
/*  - tool_count / support from the windows of every target occurrence       */
/*    (mining.py:258-275, distinct subsequences :164-183, suffixes :186-194); */
/*  - match / follow by running the literal match_at greedy (mining.py:119-  */
/*    156) for every context that could match at an anchor (all sequences   */
/*    over the signatures seen in the last k events ending with the anchor), */
/*    counting exactly what _collect_occurrences (mining.py:215-227) counts. */
/* Tables are dense as in paste_mine_desc.                                   */
/* ------------------------------------------------------------------------ */

static int64_t o_ctx_index(const int* c, int n, int S) {
  /* offset of length-n contexts = S + S^2 + ... + S^(n-1), then base-S digits */
  int64_t off = 0, p = 1, v = 0;
  int i;
  for (i = 1; i < n; ++i) { p *= S; off += p; }
  for (i = 0; i < n; ++i) v = v * S + c[i];
  return off + v;
}

/* literal match_at on a signature stream (anchored subsequence / suffix) */
static int o_match_at(const int* st, int anchor, const int* ctx, int n, int k, int relation) {
  int lo, j, pos, start, i;
  if (n == 0 || st[anchor] != ctx[n - 1]) return 0;
  if (relation == PASTE_REL_SUFFIX) {
    start = anchor - n + 1;
    if (start < 0) return 0;
    for (i = 0; i < n; ++i)
      if (st[start + i] != ctx[i]) return 0;
    return 1;
  }
  lo = anchor - k + 1;
  if (lo < 0) lo = 0;
  j = n - 2;
  pos = anchor - 1;
  while (j >= 0 && pos >= lo) {
    if (st[pos] == ctx[j]) --j;
    --pos;
  }
  return j < 0;
}

int oracle_mine_counts(const int32_t* tokens, int64_t n_tokens, int S, int k, int relation,
                       uint64_t* tool_count, uint64_t* support, uint64_t* match,
                       uint64_t* follow) {
  const int T = (S + 1) / 2;
  int64_t n_ctx = 0, p = 1, i0, i;
  int q;
  for (q = 1; q <= k; ++q) { p *= S; n_ctx += p; }
  i0 = 0;
  while (i0 < n_tokens) { /* one stream */
    int64_t i1 = i0 + 1;
    int L, j, a;
    int* st;
    while (i1 < n_tokens && !(tokens[i1] & (int32_t)0x80000000)) ++i1;
    L = (int)(i1 - i0);
    st = (int*)malloc(sizeof(int) * (size_t)L);
    for (i = 0; i < L; ++i) st[i] = (int)(tokens[i0 + i] & 0x7fffffff);
    /* targets: windows of the <= k events before j */
    for (j = 0; j < L; ++j) {
      const int tool = st[j] >> 1;
      const int lo = j - k < 0 ? 0 : j - k;
      const int wl = j - lo;
      tool_count[tool] += 1;
      if (relation == PASTE_REL_SUFFIX) {
        int s;
        for (s = lo; s < j; ++s) support[(int64_t)tool * n_ctx + o_ctx_index(st + s, j - s, S)] += 1;
      } else {
        /* distinct subsequences: collect all, dedupe by index */
        int64_t seen[64];
        int ns = 0, mask, b;
        for (mask = 1; mask < (1 << wl); ++mask) {
          int c[8], len = 0, dup = 0;
          int64_t idx;
          for (b = 0; b < wl; ++b)
            if (mask & (1 << b)) c[len++] = st[lo + b];
          idx = o_ctx_index(c, len, S);
          for (b = 0; b < ns; ++b) dup |= seen[b] == idx;
          if (dup) continue;
          seen[ns++] = idx;
          support[(int64_t)tool * n_ctx + idx] += 1;
        }
      }
    }
    /* anchors: every candidate context over the signatures of the last k
     * events that ends with the anchor, tested with the literal match_at */
    for (a = 0; a < L; ++a) {
      int alpha[8], na = 0, s, d, n;
      const int lo = a - k + 1 < 0 ? 0 : a - k + 1;
      const int lo2 = relation == PASTE_REL_SUFFIX ? (a - k + 1 < 0 ? 0 : a - k + 1) : lo;
      for (s = lo2; s < a; ++s) {
        int dup = 0;
        for (d = 0; d < na; ++d) dup |= alpha[d] == st[s];
        if (!dup) alpha[na++] = st[s];
      }
      for (n = 1; n <= k; ++n) {
        /* all sequences of length n-1 over alpha, then the anchor */
        int64_t combos = 1, cidx;
        for (d = 0; d < n - 1; ++d) combos *= na;
        for (cidx = 0; cidx < combos; ++cidx) {
          int c[8];
          int64_t v = cidx;
          for (d = n - 2; d >= 0; --d) { c[d] = alpha[v % (na ? na : 1)]; v /= (na ? na : 1); }
          c[n - 1] = st[a];
          if (!o_match_at(st, a, c, n, k, relation)) continue;
          {
            const int64_t ci = o_ctx_index(c, n, S);
            match[ci] += 1;
            if (a + 1 < L) follow[ci * T + (st[a + 1] >> 1)] += 1;
          }
        }
      }
    }
    free(st);
    i0 = i1;
  }
  return PASTE_OK;
}

/* The same counts over n_threads chunks of the stream, each cut at a stream
 * start (streams never share a window or a match, mining.py:219-226), into
 * per-thread tables that are summed: the counting above, only partitioned. */
int oracle_mine_counts_mt(const int32_t* tokens, int64_t n_tokens, int S, int k, int relation,
                          uint64_t* tool_count, uint64_t* support, uint64_t* match,
                          uint64_t* follow, int n_threads) {
  const int T = (S + 1) / 2;
  int64_t n_ctx = 0, p = 1, *cut;
  int q, t, rc = PASTE_OK;
  uint64_t* part;
  size_t per;
  if (n_threads < 2 || n_tokens < 2)
    return oracle_mine_counts(tokens, n_tokens, S, k, relation, tool_count, support, match, follow);
  for (q = 1; q <= k; ++q) { p *= S; n_ctx += p; }
  per = (size_t)T + (size_t)T * n_ctx + (size_t)n_ctx + (size_t)n_ctx * T;
  cut = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_threads + 1));
  part = (uint64_t*)calloc(per * (size_t)n_threads, sizeof(uint64_t));
  if (!cut || !part) { free(cut); free(part); return PASTE_ERR_INVALID; }
  for (t = 0; t <= n_threads; ++t) {
    int64_t c = n_tokens * t / n_threads;
    while (c > 0 && c < n_tokens && !(tokens[c] & (int32_t)0x80000000)) ++c;
    cut[t] = t == n_threads ? n_tokens : c;
  }
#pragma omp parallel for num_threads(n_threads) schedule(static, 1)
  for (t = 0; t < n_threads; ++t) {
    uint64_t* b = part + per * (size_t)t;
    int64_t lo = cut[t], hi = cut[t + 1];
    if (hi <= lo) continue; /* empty chunk */
    if (oracle_mine_counts(tokens + lo, hi - lo, S, k, relation, b, b + T, b + T + (size_t)T * n_ctx,
                           b + T + (size_t)T * n_ctx + n_ctx) != PASTE_OK)
      rc = PASTE_ERR_INVALID;
  }
  {
    int64_t i;
#pragma omp parallel for num_threads(n_threads) schedule(static)
    for (i = 0; i < (int64_t)per; ++i) {
      uint64_t s = 0;
      for (t = 0; t < n_threads; ++t) s += part[per * (size_t)t + (size_t)i];
      if (i < T) tool_count[i] += s;
      else if (i < T + (int64_t)T * n_ctx) support[i - T] += s;
      else if (i < T + (int64_t)T * n_ctx + n_ctx) match[i - T - (int64_t)T * n_ctx] += s;
      else follow[i - T - (int64_t)T * n_ctx - n_ctx] += s;
    }
  }
  free(cut);
  free(part);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* greedy_speculative_selection (scheduling.py:242-258): sort by            */
/* (-U, -p, id), U = (p * benefit) / (cost * duration); take while cost fits */
/* both slack and budget.                                                    */
/* ------------------------------------------------------------------------ */
typedef struct {
  double u, p;
  int64_t id;
  int32_t cost, idx;
} o_job;

static int o_job_cmp(const void* a_, const void* b_) {
  const o_job* a = (const o_job*)a_;
  const o_job* b = (const o_job*)b_;
  if (a->u != b->u) return a->u > b->u ? -1 : 1; /* -U ascending */
  if (a->p != b->p) return a->p > b->p ? -1 : 1; /* -p ascending */
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx ? 1 : 0); /* sorted() is stable */
}

int64_t oracle_greedy(int64_t n, const double* p, const double* benefit, const double* duration,
                      const int32_t* cost, const int64_t* id, int64_t slack, int64_t budget,
                      int32_t* selected) {
  o_job* jobs = (o_job*)malloc(sizeof(o_job) * (size_t)(n > 0 ? n : 1));
  int64_t i, n_sel = 0, r = slack, b = budget;
  for (i = 0; i < n; ++i) {
    jobs[i].u = (p[i] * benefit[i]) / ((double)cost[i] * duration[i]);
    jobs[i].p = p[i];
    jobs[i].id = id[i];
    jobs[i].cost = cost[i];
    jobs[i].idx = (int32_t)i;
  }
  qsort(jobs, (size_t)n, sizeof(o_job), o_job_cmp);
  for (i = 0; i < n; ++i)
    if (jobs[i].cost <= r && jobs[i].cost <= b) {
      selected[n_sel++] = jobs[i].idx;
      r -= jobs[i].cost;
      b -= jobs[i].cost;
    }
  free(jobs);
  return n_sel;
}

/* ------------------------------------------------------------------------ */
/* candidate_paths (mappings.py:237-266) over tapes: pre-order visit of at   */
/* most node_budget nodes, scalar leaves equal to the target (values_equal,  */
/* events.py:125-130: same type class, same canonical bytes, not NaN).       */
/* ------------------------------------------------------------------------ */
int oracle_leaf_scan(const paste_leaf_scan_desc* d, int n_threads) {
  int64_t q;
#pragma omp parallel for num_threads(n_threads > 0 ? n_threads : 1) schedule(dynamic, 64)
  for (q = 0; q < d->n_queries; ++q) {
    const paste_event_ref ref = d->refs[d->event[q]];
    const paste_tape_node* root = &d->nodes[ref.node_base];
    const int64_t total = root->type >= PASTE_T_LIST ? root->b : 1;
    const int64_t limit = total < d->node_budget ? total : d->node_budget;
    const int tt = d->target_type[q];
    const uint8_t* tb = d->target_bytes + d->target_off[q];
    const int64_t tl = d->target_off[q + 1] - d->target_off[q];
    const int64_t cap = d->out_off[q + 1] - d->out_off[q];
    int64_t i, n_out = 0;
    for (i = 0; i < limit; ++i) {
      const paste_tape_node* nd = &d->nodes[ref.node_base + i];
      int eq = 0;
      if (nd->type < PASTE_T_LIST && nd->type == tt && !d->target_nan[q] && !(nd->flags & PASTE_F_NAN)) {
        if (nd->type <= PASTE_T_TRUE) {
          eq = 1;
        } else {
          const uint8_t* b = d->bytes + ref.byte_base + nd->a;
          int64_t len = nd->b;
          if (nd->type == PASTE_T_STR && (nd->flags & PASTE_F_NFC)) {
            const uint8_t* x = b + nd->b;
            len = (int64_t)x[0] | ((int64_t)x[1] << 8) | ((int64_t)x[2] << 16) | ((int64_t)x[3] << 24);
            b = x + 4;
          }
          eq = len == tl && memcmp(b, tb, (size_t)len) == 0;
        }
      }
      if (eq) {
        if (n_out < cap) d->out_nodes[d->out_off[q] + n_out] = (int32_t)i;
        ++n_out;
      }
    }
    d->n_out[q] = n_out;
    d->truncated[q] = total > d->node_budget;
  }
  return PASTE_OK;
}
