/*
 * paste.h -- C ABI of libpaste.so, the B200 (sm_100a) engine for the
 * data-parallel core of PASTE (arXiv 2603.18897).
 *
 * The reference (spectool, /root/reference/pkg/src/spectool) is a pure-Python
 * library with no FFI layer; its drop-in surface is the Python API re-exported
 * in spectool/__init__.py:9-90.  The Python package paper_2603_18897_b200
 * mirrors that API and binds the entry points below with ctypes
 * (paper_2603_18897_b200/_native.py).  Each entry point names the reference
 * function(s) whose computation it replaces.
 *
 * Conventions
 *   - every pointer inside a *_desc / *_out struct is a DEVICE pointer
 *     (caller-owned, e.g. torch tensors); the structs themselves live in host
 *     memory and are read during the call only.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); calls are
 *     asynchronous with respect to the host unless stated otherwise.
 *   - return value: PASTE_OK (0) or a negative error class; the message of
 *     the last failure on the calling thread is available from
 *     paste_last_error().
 *   - no pointer is retained past the call.
 */
#ifndef PASTE_H
#define PASTE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PASTE_OK 0
#define PASTE_ERR_INVALID (-1)     /* bad argument (maps to ValueError)            */
#define PASTE_ERR_CUDA (-2)        /* CUDA runtime failure (maps to RuntimeError)  */
#define PASTE_ERR_UNSUPPORTED (-3) /* outside the engine's envelope                */

#define PASTE_ABI_VERSION 1

/* ---------------------------------------------------------------------- */
/* Payload tapes (see paper_2603_18897_b200/tape.py)                        */
/* ---------------------------------------------------------------------- */

enum {
  PASTE_T_NULL = 0, PASTE_T_FALSE = 1, PASTE_T_TRUE = 2, PASTE_T_INT = 3,
  PASTE_T_FLOAT = 4, PASTE_T_STR = 5, PASTE_T_LIST = 6, PASTE_T_DICT = 7
};
enum { PASTE_F_NFC = 1, PASTE_F_FLOATSRC = 2, PASTE_F_NAN = 4,
       PASTE_F_ASCII = 8 /* scalar bytes all < 0x80 (optional hint; absent = scan) */ };

typedef struct {
  uint8_t type;   /* PASTE_T_*                                                */
  uint8_t flags;  /* PASTE_F_*                                                */
  uint16_t pad;
  int32_t key;    /* interned key inside the parent dict, -1 otherwise        */
  uint32_t a;     /* container: #children      | scalar: byte offset          */
  uint32_t b;     /* container: subtree nodes  | scalar: byte length          */
} paste_tape_node; /* 16 bytes */

/* Event payload directory entry: where one event's tape starts.            */
typedef struct {
  int64_t node_base;
  int64_t byte_base;
} paste_event_ref;

/* ---------------------------------------------------------------------- */
/* Compiled pattern pool (PoolImage, paper_2603_18897_b200/packing.py)      */
/* ---------------------------------------------------------------------- */

enum { PASTE_REL_ANCHORED = 0, PASTE_REL_SUFFIX = 1 };       /* mining.py:42-51 */
enum { PASTE_X_PATH = 0, PASTE_X_FALLBACK = 1, PASTE_X_FORMAT = 2 }; /* mappings.py:47-89 */
enum { PASTE_PF_HAS_MAPPING = 1, PASTE_PF_STRUCT_ERR = 2 };

typedef struct {
  int32_t ctx_off;     /* into ctx_sig                                        */
  int32_t ctx_len;
  int32_t target_tool; /* tool id (sig >> 1)                                  */
  int32_t bind_off;    /* into bindings                                       */
  int32_t n_bind;
  int32_t flags;       /* PASTE_PF_*                                          */
  double p;            /* PatternTuple.p                                      */
} paste_pattern;       /* 32 bytes */

typedef struct {
  int32_t kind;       /* PASTE_X_*                                           */
  int32_t ctx_pos;    /* PathLookup.ctx_pos / IndexedFallback.ctx_pos / hole  */
  int32_t step_off;   /* path (PATH, FORMAT hole) or path_prefix (FALLBACK)   */
  int32_t step_cnt;
  int32_t suf_off;    /* FALLBACK path_suffix                                 */
  int32_t suf_cnt;
  int32_t start_index;/* FALLBACK start_index (clamped; <0 never resolves)    */
  int32_t fail_tool;  /* FALLBACK fail_tool id, -1 = unknown tool             */
} paste_binding;      /* 32 bytes */

/* A path step is a pair (kind, value): kind 0 = dict key id, 1 = list index
 * (negative / out of int32 range = never resolves).                         */
typedef struct {
  int32_t n_patterns;
  int32_t n_bucket_sigs;   /* buckets exist for sig < n_bucket_sigs           */
  int32_t k;               /* MiningConfig.k of the pool                      */
  int32_t relation;        /* PASTE_REL_*                                     */
  int32_t max_ctx;         /* longest context                                 */
  int32_t max_bindings;
  const paste_pattern* patterns;
  const paste_binding* bindings;
  const int32_t* ctx_sig;
  const int32_t* steps;        /* 2 x int32 per step                          */
  const int32_t* bucket_off;   /* [n_bucket_sigs + 1]                         */
  const int32_t* bucket_pat;   /* pattern ids, static rank (-p, pattern_id)   */
  const uint8_t* bucket_scan_all; /* 1 = bucket holds a struct-error pattern  */
  /* optional match table (paste_build_match_table): NULL = scan buckets.
   * Valid for requests with max_candidates <= mt_k and the same gather
   * depth mt_g = min(k | max_ctx, window capacity).                         */
  const void* match_table;
  int32_t mt_k;
  int32_t mt_g;
} paste_pool_desc;

/* Per-tool admission tables (policy.py:207-244, scheduling.py:218-219).    */
typedef struct {
  int32_t enabled;          /* 0 = predict only                               */
  int32_t n_tools;
  const uint8_t* allow;     /* [n_tools] ToolRule.allow                       */
  const uint8_t* max_level; /* [n_tools] 1 warm_only, 2 dry_run, 3 full       */
  const double* benefit;    /* [n_tools] benefit_of(tool), e.g. EWMA duration */
} paste_admit_desc;

/* ---------------------------------------------------------------------- */
/* Live session windows (PredictionWindow, prediction.py:40-58)             */
/* ---------------------------------------------------------------------- */

typedef struct {
  int64_t n_sessions;
  int32_t capacity;            /* W (ring slots per session)                  */
  int32_t slot_major;          /* 0: tok/evt are [n][W]; 1: [W][n] (sessions
                                  stepping together touch contiguous slots)  */
  int32_t* tok;                /* ring: sig id, -1 = LLM step                 */
  int32_t* evt;                /* ring: event index into refs                 */
  int64_t* count;              /* [n] events observed so far                  */
  const paste_tape_node* nodes;
  const uint8_t* bytes;
  paste_event_ref* refs;       /* event directory (written by observe)        */
  /* optional observe-before-predict: session s first observes one new event
   * (token new_tok[s]); it becomes event new_evt_base + s and its directory
   * entry is new_ref[s] with byte_base taken relative to new_byte_base.     */
  const int32_t* new_tok;      /* [n] or NULL                                 */
  const paste_event_ref* new_ref; /* [n] (or NULL when new_node is given)     */
  int64_t new_evt_base;
  int64_t new_byte_base;
  /* optional stream mode (replay): windows are views into one event stream.
   * tok / evt are then the stream, count[s] (<= capacity) is window s's
   * length and window s = stream[stream_end[s] - count[s] .. stream_end[s]);
   * new_tok must be NULL.                                                  */
  const int64_t* stream_end;
  /* optional narrow observe input: node_base only (byte_base = new_byte_base),
   * 4 B/session instead of the 16-B directory entry of new_ref            */
  const int32_t* new_node;
  /* optional narrow wire form of the observe input (live-plan kernels only):
   * token u8 (255 = LLM step) and node_base u16 (byte_base = new_byte_base);
   * when set they replace new_tok / new_node                               */
  const uint8_t* new_tok8;
  const uint16_t* new_node16;
  /* optional 2-byte wire form (with new_tok8, instead of new_node16): a u8
   * node code per session and the code -> node_base table [256]; the caller
   * assigns codes to the node arrays (payload shapes) it has seen          */
  const uint8_t* new_node8;
  const int32_t* node_codes;
  /* optional 1-byte wire form (with new_tok8 alone): new_tok8 holds a u8
   * event code per session and event_codes[2 * code] is its token (-1 = LLM
   * step), event_codes[2 * code + 1] its node_base; the caller assigns codes
   * to the (token, node array) pairs it has seen                           */
  const int32_t* event_codes;
} paste_windows;

enum { PASTE_C_FULL = 0, PASTE_C_PARTIAL = 1, PASTE_C_TOOL_ONLY = 2 };

typedef struct {
  int32_t max_candidates;  /* K: per-session prediction slots                 */
  int32_t max_bindings;    /* slots per prediction in pred_arg                */
  int32_t slot_major;      /* 0: per-session records [n][K] ([n][K][B] args);
                              1: slot-major [K][n] ([K][B][n] args)           */
  int32_t pad;
  int32_t* n_pred;         /* [n]                                             */
  int32_t* pred_pat;       /* [n*K] pattern index                             */
  uint8_t* pred_comp;      /* [n*K] PASTE_C_*                                 */
  int64_t* pred_arg;       /* [n*K*B] (event << 32 | node) or -1 = UNBOUND    */
  int32_t* n_act;          /* [n]                                             */
  int16_t* act_pred;       /* [n*K] prediction slot of each action, in order  */
  uint8_t* act_level;      /* [n*K] SpecLevel                                 */
  double* act_util;        /* [n*K] expected utility p * benefit              */
  int32_t* struct_err;     /* [n] structural errors met (diagnostics)         */
} paste_predict_out;

/* ---------------------------------------------------------------------- */
/* Entry points                                                             */
/* ---------------------------------------------------------------------- */

const char* paste_last_error(void);
int paste_abi_version(void);

/* K4: batched Predictor.predict + admit.
 * Replaces prediction.py:76-118 (Predictor.predict, incl. match_at
 * mining.py:119-156 and evaluate mappings.py:207-223) and policy.py:207-244
 * (admit) for every session of the batch; when windows->new_tok is non-NULL
 * each session first observes one new event (PredictionWindow.observe,
 * prediction.py:48-49).                                                    */
int paste_predict_batch(const paste_pool_desc* pool, paste_windows* windows,
                        const paste_admit_desc* admit, paste_predict_out* out,
                        void* stream);

/* Pool compilation for K4: a match table keyed by the newest G tool tokens.
 * Which patterns match at an anchor, in which order and at which positions
 * depends only on those G tokens (match_at looks back at most k events,
 * mining.py:142), so the table stores per key the number of matches, the
 * number of structural-error matches (Predictor diagnostics) and the first
 * max_candidates matches in rank order with the matched position (age) of
 * every binding's source event.  Key = anchor + S * sum_{a>=1} code(age a)
 * * (S+1)^(a-1) with S = n_bucket_sigs and code = S for "no event / unknown
 * signature".  Entry = {int32 n_match, int32 n_err, 2 x pad} + max_candidates records
 * of 32 bytes {pid, 4-bit source age per binding, target tool,
 * n_bind | flags << 16, bind_off, pad, double p}.
 * paste_match_table_bytes returns the size, or -1 when the pool is outside
 * the table's envelope (the kernel then scans buckets).                    */
int64_t paste_match_table_bytes(const paste_pool_desc* pool, int32_t max_candidates,
                                int32_t window_capacity);
int paste_build_match_table(const paste_pool_desc* pool, int32_t max_candidates,
                            int32_t window_capacity, void* table, void* stream);

/* K4 epilogue as a standalone op: admit() over many prediction lists.
 * Replaces policy.py:207-244 (admit + _beats).  Per prediction: tool id,
 * full (1 = Completeness.FULL), probability, benefit_of(prediction) and
 * created_at; lists are CSR (list_off[n_lists+1]).  Output per list: the
 * number of actions and, in first-appearance order, the winning prediction
 * (index within its list), level and expected utility; slots are
 * list_off-aligned (at most one action per prediction).                    */
typedef struct {
  int64_t n_lists;
  const int64_t* list_off;  /* [n_lists + 1]                                 */
  const int32_t* tool;      /* [N]                                           */
  const uint8_t* full;      /* [N]                                           */
  const double* p;          /* [N]                                           */
  const double* benefit;    /* [N]                                           */
  const double* created_at; /* [N]                                           */
  int32_t* n_act;           /* [n_lists]                                     */
  int32_t* act_pred;        /* [N]                                           */
  uint8_t* act_level;       /* [N]                                           */
  double* act_util;         /* [N]                                           */
} paste_admit_lists_desc;

int paste_admit_lists(const paste_admit_desc* policy, paste_admit_lists_desc* lists,
                      void* stream);

/* ---------------------------------------------------------------------- */
/* Mining (K1 ingest, K2 count, selection; mining.py:164-292)               */
/* ---------------------------------------------------------------------- */

/* Token stream: int32 sig ids, bit 31 set on the first tool event of every
 * segment (session after inactivity splitting).  Tables are dense over
 * S = n_sigs signatures and contexts of length 1..k: context (c_1..c_n) has
 * index sum_{m<n} S^m + sum_i c_i * S^(n-i); T = S / 2 tools.             */
typedef struct {
  int32_t n_sigs;
  int32_t k;                 /* MiningConfig.k (1..6)                          */
  int32_t relation;          /* PASTE_REL_*                                    */
  int32_t pad;
  const int32_t* tokens;     /* [n_tokens] flagged token stream               */
  int64_t n_tokens;
  uint32_t* hist;            /* [(S+2)^(k+1)] (k+1)-gram histogram (zeroed)    */
  uint64_t* tool_count;      /* [T]        occurrences per tool (zeroed)       */
  uint64_t* support;         /* [T][n_ctx] window support (zeroed)             */
  uint64_t* match;           /* [n_ctx]    anchored matches (zeroed)           */
  uint64_t* follow;          /* [n_ctx][T] matches followed by the tool (zeroed)*/
} paste_mine_desc;

/* Sizes of the dense histogram and context space for (n_sigs, k).          */
int paste_mine_geometry(int32_t n_sigs, int32_t k, int64_t* n_bins, int64_t* n_ctx);
/* K2: accumulate the (k+1)-gram histogram of a token stream (adds to hist,
 * so shards can be counted into one histogram or merged by all-reduce).    */
int paste_mine_count(const paste_mine_desc* d, void* stream);
/* Expand the histogram into tool_count / support / match / follow.         */
int paste_mine_expand(const paste_mine_desc* d, void* stream);

/* Target-sliced tail for strong scaling.  support[t][*],
 * follow[*][t] and tool_count[t] only read histogram column s0 in {2t,
 * 2t+1} (the gram's last symbol = the target), and match[c] only reads the
 * grams whose last symbol is c's last symbol (the anchor).  So with the
 * columns cut into n_slices equal blocks of `slice_cols` (even, covering
 * every sig; paste_mine_slice_cols), rank r expands block r alone:
 *   paste_mine_transpose_slices: hist [window][s0] -> hist_t [s0][window]
 *     for s0 < n_slices * slice_cols (columns >= n_sigs are zero), so block
 *     r is contiguous (reduce-scatter it);
 *   paste_mine_expand_slice: expand block r (slice [col_lo, col_lo +
 *     slice_cols) of hist_t, [slice_cols][base^k]) into the zeroed tables:
 *     complete values for the block's tools and for the match of contexts
 *     whose last signature is in the block, zero elsewhere (sum the match
 *     arrays over the ranks; the other tables are disjoint).              */
int32_t paste_mine_slice_cols(int32_t n_sigs, int32_t n_slices);
int paste_mine_transpose_slices(const paste_mine_desc* d, int32_t n_slices, uint32_t* hist_t,
                                void* stream);
int paste_mine_expand_slice(const paste_mine_desc* d, const uint32_t* slice, int32_t col_lo,
                            int32_t slice_cols, void* stream);
/* Candidates (target, context) with tool_count >= sigma, support >= sigma,
 * match > 0 and follow / match >= tau (the upper bound of p for any
 * mapping): out[5*i..] = {tool, context index, support, match, follow};
 * *n_out receives the number found (only the first `cap` are written).    */
int paste_mine_select(const paste_mine_desc* d, int64_t sigma, double tau, int64_t cap,
                      uint64_t* n_out, int64_t* out, void* stream);

/* Mapping-free selection in mine()'s output order (mining.py:105-111):
 * rows (tool, context index, support, match, follow, p as f64 bits) of the
 * pairs with tool_count >= sigma, support >= sigma, match > 0 and
 * p = follow / match >= tau, sorted by (-p, -len, target, context).  *n_out
 * receives the number found (only the first `cap` are ranked and written:
 * callers retry with a larger cap when *n_out > cap).  `scratch` is device
 * memory of paste_mine_sort_scratch_bytes(cap) bytes.                      */
int64_t paste_mine_sort_scratch_bytes(int64_t cap);
int paste_mine_select_sorted(const paste_mine_desc* d, int64_t sigma, double tau, int64_t cap,
                             uint64_t* n_out, int64_t* out, void* scratch, void* stream);

/* K1 + K2 fused over a columnar trace of tool events grouped by session
 * (sessions in first-appearance order, events sorted by (t_start, seq)):
 * segments split where t_start - prev.t_end > inactivity_ms (events.py:
 * 196-252), then the (k+1)-gram histogram is accumulated into d->hist.
 * Order violations are counted in *n_unsorted (callers must reject them).  */
typedef struct {
  int64_t n_events;
  const int32_t* session;   /* [n] session index, non-decreasing             */
  const int32_t* seq;       /* [n]                                           */
  const double* t_start;    /* [n] ms                                        */
  const double* t_end;      /* [n] ms                                        */
  const int32_t* sig;       /* [n] tool signature id                         */
  double inactivity_ms;
  int32_t* tokens_out;      /* optional [n]: flagged token stream            */
  uint64_t* n_segments;     /* optional counter                              */
  uint64_t* n_unsorted;     /* optional counter                              */
} paste_columnar_desc;

int paste_mine_ingest_count(const paste_columnar_desc* c, const paste_mine_desc* d, void* stream);

/* Native (host, OpenMP) columnar ingest of a JSONL trace for mining:
 * ingest_trace (events.py:196-252) -- group by session_id in first-
 * appearance order, stable sort by (t_start, seq), split on gaps over all
 * events, keep each segment's tool events (Session.tool_events) -- written
 * as the columnar trace above with session = segment index (count it with
 * no further gap split: inactivity_ms = +inf) and sig = 2 * tool + success,
 * tools interned in sorted name order (tool_names: sorted, NUL-separated).
 * Lines missing a required field, or that Event.__post_init__ rejects
 * (t_start > t_end; a tool_call with an empty tool), are errors
 * (error_lines, 1-based; error_codes / error_seq give the reason).  Input
 * outside the parser's exact subset (escapes in ids, non-string ids,
 * non-integral seq, NaN start times, duplicate keys, unvalidated JSON,
 * other line separators) returns PASTE_ERR_UNSUPPORTED: use the host
 * ingest.  Capacities too small: PASTE_ERR_INVALID with the counts set.     */
typedef struct {
  int64_t capacity;            /* event slots in the columns below            */
  int32_t* session;
  int32_t* seq;
  double* t_start;
  double* t_end;
  int32_t* sig;
  int32_t* error_lines;        /* optional [error_capacity]                   */
  int64_t error_capacity;
  char* tool_names;            /* optional [tool_names_capacity]              */
  int64_t tool_names_capacity;
  int64_t n_events;            /* out: tool events                            */
  int64_t n_segments;          /* out                                         */
  int64_t n_errors;            /* out                                         */
  int64_t n_lines;             /* out                                         */
  int64_t reordered_sessions;  /* out                                         */
  int64_t tool_names_len;      /* out                                         */
  int32_t n_tools;             /* out                                         */
  int32_t pad;
  int32_t* error_codes;        /* optional [error_capacity]: PASTE_INGEST_*   */
  int64_t* error_seq;          /* optional [error_capacity]: the record's seq */
} paste_ingest_desc;

/* error_codes: PASTE_INGEST_MISSING | mask of the absent fields (bit i =
 * _REQUIRED_FIELDS[i]: session_id, seq, kind, tool, status, t_start_ms,
 * t_end_ms; "missing fields: ..."), PASTE_INGEST_T_ORDER ("event seq=N:
 * t_start > t_end"), PASTE_INGEST_EMPTY_TOOL ("event seq=N: tool_call with
 * empty tool_type") -- events.py:59-63,142-145.                             */
#define PASTE_INGEST_MISSING 0x100
#define PASTE_INGEST_T_ORDER 0x200
#define PASTE_INGEST_EMPTY_TOOL 0x400

int paste_ingest_jsonl(const char* text, int64_t len, double inactivity_ms, paste_ingest_desc* d);

/* Native JSONL parse feeding the DEVICE ingest (K1 general path,
 * paste_ingest_order) and device Phase II: _parse_record (events.py:
 * 165-184) for every line in parallel, with the records' payloads.
 * Output, in FILE order, one row per valid record (errors as above):
 * session = first-appearance index of session_id, sig = 2 * tool + success
 * (tools in sorted name order) or -1 for an LLM step; and, with
 * want_payloads, the record's `result` and `args` (record.get: absent =
 * null) as payload tapes (tape.py layout, canonical scalar bytes of
 * events.py:94-130: ints as digits, integral floats as int digits with
 * FLOATSRC, other floats as Python's repr, strings as UTF-8): tape 2r =
 * result of row r, 2r + 1 = its args; dict keys interned in first-seen
 * order (key_names: NUL-separated, id = position).  The grouping, sort and
 * gap split are left to the device.  Input outside the parser's exact
 * subset (see paste_ingest_jsonl, plus: payload strings with a lone
 * surrogate or a code point >= U+0300 whose NFC form needs the Unicode
 * database, duplicate keys inside a payload, nesting deeper than 512)
 * returns PASTE_ERR_UNSUPPORTED: use the host ingest.  The result is an
 * opaque host handle: query sizes, copy into caller buffers, destroy.     */
typedef struct paste_jsonl paste_jsonl;
typedef struct {
  int64_t n_rows;
  int64_t n_sessions;
  int64_t n_errors;
  int64_t n_lines;
  int64_t n_nodes;
  int64_t n_bytes;
  int64_t n_keys;
  int64_t key_names_len;
  int64_t tool_names_len;
  int32_t n_tools;
  int32_t pad;
} paste_jsonl_sizes;
typedef struct {             /* host buffers sized by paste_jsonl_sizes      */
  int32_t* session;          /* [n_rows]                                     */
  int32_t* seq;
  double* t_start;
  double* t_end;
  int32_t* sig;
  int32_t* error_lines;      /* [n_errors]                                   */
  int32_t* error_codes;
  int64_t* error_seq;
  char* tool_names;          /* [tool_names_len]                             */
  paste_tape_node* nodes;    /* [n_nodes]      (payloads only)               */
  uint8_t* bytes;            /* [n_bytes]                                    */
  paste_event_ref* refs;     /* [2 * n_rows]                                 */
  char* key_names;           /* [key_names_len]                              */
} paste_jsonl_out;

int paste_jsonl_parse(const char* text, int64_t len, int32_t want_payloads, paste_jsonl** out);
int paste_jsonl_sizes_of(const paste_jsonl* h, paste_jsonl_sizes* s);
int paste_jsonl_copy(const paste_jsonl* h, const paste_jsonl_out* o);
void paste_jsonl_destroy(paste_jsonl* h);
/* Same, in two passes: the columnar pass writes one staged word per event
 * (4 B) to `stage`; a second pass sends the cold grams to L2 into 8
 * histogram replicas (a hot gram's updates spread over 8 addresses), which
 * are then folded into d->hist.  The scattered updates no longer contend
 * with the columnar stream.  `stage` is device memory of
 * paste_mine_stage_bytes(n_events, n_sigs, k) bytes (16-byte aligned);
 * NULL falls back to the single pass.                                      */
int64_t paste_mine_stage_bytes(int64_t n_events, int32_t n_sigs, int32_t k);
int paste_mine_ingest_count_staged(const paste_columnar_desc* c, const paste_mine_desc* d,
                                   void* stage, int64_t stage_bytes, void* stream);

/* K1 general path: ingest_trace's grouping, stable sort, reorder tally and
 * gap split (events.py:196-252, _split_on_gaps :243-252) on the device, for
 * columnar traces in ARRIVAL order (the order records were read), with
 * every event of every kind.  Replaces the host-only grouping/sort of
 * ingest_trace (events.py:212-241) on the columnar path.
 *   session: [n] session id in [0, n_sessions).  Groups are emitted in id
 *            order: pass first-appearance ids (the order ingest_trace's
 *            `order` list holds) to reproduce the reference.  Unused ids
 *            are allowed and give no segment.
 *   sig:     [n] tool signature, or -1 for an LLM step (LLM steps take
 *            part in the sort and the gap split but are not written out).
 * Each session's events are stably sorted by (t_start, seq) (-0.0 == 0.0,
 * arrival order breaks ties, as Python's sorted); a session counts as
 * reordered when its seq list changed; a new segment starts where
 * t_start - prev.t_end > inactivity_ms.  Output: the columnar mining trace
 * of paste_mine_ingest_count (tool events only, session = global segment
 * index, segments numbered in (session id, segment) order, LLM-only
 * segments included in the numbering) -- count it with inactivity_ms = +inf.
 * Device-side results: *n_out tool events, *n_segments, *reordered, and
 * *status (PASTE_ORDER_NAN_T: a NaN t_start, whose Python sort order is
 * undefined -- the caller must use the host ingest; PASTE_ORDER_BAD_SESSION:
 * an id outside [0, n_sessions)).  `order` (optional, [n]) receives the
 * arrival index of every event in sorted order (payload gathers).
 * Requires n_events < 2^31.  `scratch`: paste_ingest_order_scratch_bytes.  */
typedef struct {
  int64_t n_events;
  int32_t n_sessions;
  int32_t pad;
  const int32_t* session;
  const int32_t* seq;
  const double* t_start;
  const double* t_end;
  const int32_t* sig;
  double inactivity_ms;
  int32_t* out_session;     /* [n] capacity                                  */
  int32_t* out_seq;
  double* out_t_start;
  double* out_t_end;
  int32_t* out_sig;
  int32_t* order;           /* optional [n]                                  */
  int32_t* out_tok;         /* optional [n]: flagged token stream of the
                               output (sig, bit 31 on a segment's first tool
                               event) for paste_mine_count / occurrences     */
  int64_t* n_out;           /* device scalars                                */
  int64_t* n_segments;
  int64_t* reordered;
  int64_t* status;
} paste_order_desc;

#define PASTE_ORDER_NAN_T 1
#define PASTE_ORDER_BAD_SESSION 2

int64_t paste_ingest_order_scratch_bytes(int64_t n_events, int32_t n_sessions);
int paste_ingest_order(const paste_order_desc* d, void* scratch, int64_t scratch_bytes,
                       void* stream);

/* Phase II occurrence collection: _collect_occurrences (mining.py:215-227)
 * for many candidates in one pass, keeping the followed occurrences whose
 * next event has the candidate's target tool -- the `occ` list mine()
 * hands to infer_mapping / mapping_holds (:277-285).  Replaces the host's
 * per-candidate rescan of every stream.
 * For every anchor a of the flagged token stream (bit 31 = first event of a
 * session stream, token = 2 * tool + success) whose next token is in the
 * same stream, the candidates of bucket (sig(a), tool(a + 1)) are matched
 * with match_at (:119-156: last context sig == the anchor's; anchored
 * rightmost embedding inside the k events ending at a, or the contiguous
 * suffix slice), never across a stream boundary.  Candidate c's
 * occurrences land in slots [off[c], off[c+1]) -- off is the exclusive scan
 * of the candidates' follow counts from the mining tables, which count
 * exactly these occurrences -- in no particular order: anchor[slot] = a,
 * picked[slot * kmax + j] = stream position of matched event j (the
 * history is [picked[slot * kmax], a]).  `cursor` ([n_cand], zeroed by the
 * caller) and *overflow (emissions past a candidate's range; must stay 0)
 * are device memory.  Sort slots by (candidate, anchor) with
 * paste_ingest_order (session = candidate, t_start = anchor) for stream
 * order.                                                                   */
typedef struct {
  int64_t n_tokens;
  const int32_t* tok;
  int32_t n_cand;
  int32_t k;                /* MiningConfig.k                                */
  int32_t relation;         /* 0 anchored subsequence, 1 contiguous suffix   */
  int32_t kmax;             /* row width of ctx / picked (>= every ctx_len)  */
  int32_t n_sigs;
  int32_t n_tools;
  const int32_t* ctx;       /* [n_cand * kmax] context sigs                  */
  const int32_t* ctx_len;   /* [n_cand]                                      */
  const int32_t* bucket_off;/* [n_sigs * n_tools + 1] by (last sig, target)  */
  const int32_t* bucket;    /* candidate ids                                 */
  const int64_t* off;       /* [n_cand + 1]                                  */
  int64_t* cursor;          /* [n_cand]                                      */
  int64_t* anchor;          /* [off[n_cand]]                                 */
  int32_t* picked;          /* [off[n_cand] * kmax]                          */
  uint64_t* overflow;
} paste_occ_desc;

int paste_mine_occurrences(const paste_occ_desc* d, void* stream);

/* ---------------------------------------------------------------------- */
/* canonical_arg_hash (events.py:94-122) on the device                      */
/* ---------------------------------------------------------------------- */

/* blake2b-128 of canonical_json(value) for n payload tapes (one value per
 * directory entry).  key_bytes / key_off hold the NFC form of every interned
 * key (UTF-8), key_rank its rank in code-point order (equal NFC forms share
 * a rank).  unsure[i] = 1 when the value is left to the host: two keys of
 * one dict with the same NFC form, a lone surrogate (the reference's
 * .encode raises), nesting deeper than 32, a dict wider than 256 keys.     */
typedef struct {
  int64_t n;
  const paste_tape_node* nodes;
  const uint8_t* bytes;
  const paste_event_ref* refs;   /* [n]                                      */
  const uint8_t* key_bytes;
  const int64_t* key_off;        /* [n_keys + 1]                             */
  const int32_t* key_rank;       /* [n_keys]                                 */
  uint8_t* digest;               /* [n][16]                                  */
  uint8_t* unsure;               /* [n]                                      */
} paste_hash_desc;

int paste_canonical_hash(const paste_hash_desc* d, void* stream);

/* Scheduler cache keys of the admitted actions of one live step
 * (scheduling.py:464-480: key = (tool, canonical_arg_hash(prediction.args))
 * for every non-WARM_ONLY action).  Reads paste_predict_batch's records;
 * writes keys[slot][16] for action slot (same addressing as act_pred) and
 * key_state[slot]: 0 = key written, 1 = WARM_ONLY (no argument key), 2 =
 * unsure (non-ASCII FormatTemplate text, NFC-colliding names, deep / wide
 * values: hash the decoded arguments on the host).  Keys of the payload
 * and the arg names come from one key table (NFC bytes + code-point ranks,
 * as for paste_canonical_hash); bind_key / fmt / fmt_bytes as for
 * paste_replay_score.                                                     */
typedef struct {
  int64_t n_sessions;
  paste_pool_desc pool;
  paste_predict_out out;
  const paste_tape_node* nodes;
  const uint8_t* bytes;
  const paste_event_ref* refs;
  const uint8_t* key_bytes;
  const int64_t* key_off;
  const int32_t* key_rank;
  const int32_t* bind_key;   /* [n_bindings] key id of each binding's arg name */
  const int32_t* fmt;        /* [n_bindings][5] FormatTemplate rows            */
  const uint8_t* fmt_bytes;
  uint8_t* keys;             /* [n * K][16]                                     */
  uint8_t* key_state;        /* [n * K]                                         */
} paste_action_keys_desc;

int paste_action_keys(const paste_action_keys_desc* d, void* stream);

/* ---------------------------------------------------------------------- */
/* A16: admitted actions -> scheduler jobs (scheduling.py:464-511, 59-60)   */
/* ---------------------------------------------------------------------- */

/* Admitted actions in batch order (sessions in order, each session's
 * actions in admit order), as Scheduler.submit_speculative_batch feeds them
 * to _admit_action.                                                        */
typedef struct {
  int64_t n_actions;
  const int32_t* tool;        /* [n] tool id                                   */
  const uint8_t* level;       /* [n] SpecLevel: 1 warm_only, 2 dry_run, 3 full */
  const double* p;            /* [n] prediction.probability                    */
  const uint8_t* key;         /* [n][16] canonical_arg_hash(args) digest (16-B
                                 aligned; ignored for WARM_ONLY)               */
  int32_t n_tools;
  int32_t pad;
  const double* mean;         /* [n_tools] EstimateBook.duration(tool)         */
  const int32_t* cost;        /* [n_tools] EstimateBook.cost(tool)             */
  double warm_fraction;       /* EstimateBook.warm_fraction                    */
  int64_t r_total;            /* ResourceState.r_total (cost > r_total: drop)  */
  int64_t id_base;            /* the scheduler's next job id                   */
} paste_actions_desc;

/* Job columns (the paste_select_desc inputs), in batch order.              */
typedef struct {
  double* p;                  /* [<= n] Job.p                                  */
  double* benefit;            /* [<= n] Job.benefit_ms                         */
  double* duration;           /* [<= n] Job.duration_est_ms                    */
  int32_t* cost;              /* [<= n] Job.cost                               */
  int64_t* id;                /* [<= n] Job.id                                 */
  int64_t* action;            /* [<= n] source action index, or NULL           */
  int64_t* n_jobs;            /* [1] jobs written                              */
  int64_t* next_id;           /* [1] id_base + ids consumed                    */
} paste_jobs_out;

/* _admit_action over a batch into a fresh scheduler: terms per level
 * (WARM_ONLY T = wf*mean, d = max(wf*mean, 1e-9); DRY_RUN T = wf*mean,
 * d = max(mean, 1e-9); FULL T = mean, d = max(mean, 1e-9)), in-batch key
 * coalescing (first action of a key wins), ids in batch order, cost >
 * r_total dropped after taking an id.  Synchronous.                        */
int64_t paste_action_jobs_scratch_bytes(int64_t n_actions);
int paste_action_jobs(const paste_actions_desc* a, paste_jobs_out* j, void* scratch,
                      int64_t scratch_bytes, void* stream);

/* A live step's K-slot records -> action columns in batch order (tool =
 * pattern target, p = pattern p, key copied from paste_action_keys' output
 * slot when slot_keys is non-NULL).  Stream-ordered; *n_actions on device. */
typedef struct {
  int64_t n_sessions;
  paste_pool_desc pool;
  paste_predict_out out;
  const uint8_t* slot_keys;   /* [n*K][16] paste_action_keys output, or NULL   */
  int32_t* tool;              /* [<= n*K]                                      */
  uint8_t* level;
  double* p;
  uint8_t* key;               /* [<= n*K][16] (when slot_keys)                 */
  int64_t* session;           /* [<= n*K] session of each action               */
  int32_t* slot;              /* [<= n*K] record slot of each action           */
  int64_t* n_actions;         /* [1]                                           */
} paste_live_actions_desc;

int64_t paste_live_actions_scratch_bytes(int64_t n_sessions);
int paste_live_actions(const paste_live_actions_desc* l, void* scratch, int64_t scratch_bytes,
                       void* stream);

/* ---------------------------------------------------------------------- */
/* K6: admission selection (scheduling.py:59-60, 242-258)                   */
/* ---------------------------------------------------------------------- */

typedef struct {
  int64_t n_jobs;
  const double* p;          /* [n] Job.p                                      */
  const double* benefit;    /* [n] Job.benefit_ms                             */
  const double* duration;   /* [n] Job.duration_est_ms                        */
  const int32_t* cost;      /* [n] Job.cost (>= 1)                            */
  const int64_t* id;        /* [n] Job.id                                     */
  int32_t* selected;        /* [<= min(slack, budget)] chosen job indices, in
                               selection order                                */
  int64_t* n_selected;      /* [1]                                            */
} paste_select_desc;

/* greedy_speculative_selection: jobs in ascending (-U, -p, id) with
 * U = (p * benefit) / (cost * duration), taken while cost fits both the
 * remaining slack and budget.  Synchronous (returns after the result is
 * written).  min(slack, budget) <= 64: per-cost-class radix select + on-chip
 * sort; larger caps (or > 4,096 tied candidates): full device sort path.   */
int64_t paste_select_scratch_bytes(int64_t n_jobs);
int paste_select_greedy(paste_select_desc* d, int64_t slack, int64_t budget, void* scratch,
                        int64_t scratch_bytes, void* stream);

/* Stage-2 preemption victim (scheduling.py:571-578): index of the job with
 * the smallest (U, -id), -1 for no jobs (selected / n_selected unused).
 * scratch: >= 4 bytes of device memory.  Synchronous.                      */
int paste_select_victim(const paste_select_desc* d, int32_t* out_idx, void* scratch,
                        void* stream);

/* ---------------------------------------------------------------------- */
/* K5: leaf scan and expression resolution over payload tapes               */
/* ---------------------------------------------------------------------- */

/* candidate_paths (mappings.py:237-266) for many (payload, target) pairs:
 * the first node_budget nodes of each payload (pre-order = tape order) are
 * compared with the target scalar (values_equal, events.py:125-130); the
 * matching node indices are written in order (at most out_off[q+1] -
 * out_off[q] of them; n_out[q] is the full count).  target_type is the
 * tape type of the target scalar, -1 for a container (never equal);
 * target bytes are its canonical bytes (NFC for strings).                  */
typedef struct {
  int64_t n_queries;
  int64_t node_budget;
  const paste_tape_node* nodes;
  const uint8_t* bytes;
  const paste_event_ref* refs;
  const int32_t* event;        /* [n] payload (event) index                   */
  const int32_t* target_type;  /* [n]                                         */
  const uint8_t* target_nan;   /* [n]                                         */
  const int64_t* target_off;   /* [n+1] into target_bytes                     */
  const uint8_t* target_bytes;
  const int64_t* out_off;      /* [n+1] into out_nodes                        */
  int32_t* out_nodes;
  int64_t* n_out;              /* [n]                                         */
  uint8_t* truncated;          /* [n]                                         */
} paste_leaf_scan_desc;

int paste_leaf_scan(const paste_leaf_scan_desc* d, void* stream);
/* The same for queries grouped by payload shape (shape-interned tapes):
 * queries whose payloads share a node array and whose targets share type
 * and canonical length form a group (group[q]; group_rep[g] = any member).
 * The group's candidate nodes are listed once (in pre-order, within the
 * budget), then each query compares only those with its own bytes.
 * scratch: paste_leaf_scan_shared_bytes(n_groups, node_budget) bytes.      */
int64_t paste_leaf_scan_shared_bytes(int64_t n_groups, int64_t node_budget);
int paste_leaf_scan_shared(const paste_leaf_scan_desc* d, const int32_t* group, int64_t n_groups,
                           const int32_t* group_rep, void* scratch, void* stream);

/* evaluate()'s resolution (mappings.py:143-194) of one binding per query
 * against an explicit source event; for IndexedFallback the history tokens
 * after src_pos are scanned for FAIL events of fail_tool (-1 tokens mark the
 * source event itself and are skipped).  result[q] = node index or -1.     */
typedef struct {
  int64_t n_queries;
  const paste_binding* bindings; /* [n]                                       */
  const int32_t* steps;
  const paste_tape_node* nodes;
  const paste_event_ref* refs;
  const int32_t* src_event;      /* [n]                                       */
  const int32_t* hist_off;       /* [n+1]                                     */
  const int32_t* hist_tok;       /* sig per history event, -1 = source        */
  const int32_t* src_pos;        /* [n] source position in its history, -1    */
  int64_t* result;               /* [n]                                       */
} paste_resolve_desc;

int paste_resolve(const paste_resolve_desc* d, void* stream);

/* Live-path record compaction: the K-slot records of paste_predict_batch
 * -> narrow CSR streams in session order (decoupled look-back scan).
 * Capacities: pred/act n*K, arg n*K*B.  Streams (element widths per
 * `format`):
 *   hdr  u16 n_pred | n_act << 8          (PASTE_CF_HDR8: u8 n_pred | n_act << 4)
 *   pred u16 pattern | completeness << 14  (PASTE_CF_PRED8: u8 pattern | completeness << 6)
 *   arg  u32 region << 27 | node           (PASTE_CF_ARG16: u16 region << 11 | node)
 *        for the n_bind references of mapped predictions only, the source
 *        event being region * n_sessions + session (the live table's event
 *        ids); all-ones = unresolved
 *   act  u8  slot | level << 5
 * The expected utility of an action is p(pattern) * benefit(tool)
 * (policy.py:224-232), which the host redoes exactly, so it is not shipped.
 * totals = {predictions, arguments, actions, refs outside the chosen arg
 * form (0 expected: else re-fetch the full records), structural errors}.
 * Requires max_candidates <= 31 and n_patterns <= 16384; HDR8 needs
 * max_candidates <= 15, PRED8 n_patterns <= 64.
 * PASTE_CF_ENTRY16 (paste_predict_compact only): the pred stream instead
 * holds one u16 per session, the session's match-table key (0xFFFF = no
 * entry, no predictions).  The predictions are the first n_pred records of
 * that entry (paste_build_match_table), so the host expands them from its
 * copy of the table; completeness follows from the pattern (no mapping =
 * TOOL_ONLY) and the arg stream (an all-ones reference = PARTIAL).
 * PASTE_CF_KEYS (with PASTE_CF_ENTRY16, paste_predict_live_compact only):
 * the hdr and act streams are not written either -- a session's counts and
 * actions follow from its key's live-plan entry (paste_build_live_plan: the
 * same admit decisions) and its arg stream (an unresolved reference makes
 * the prediction PARTIAL, which admits it at the entry's partial level); the
 * host expands them from its copy of the plan.  Streams: key + arg.
 * PASTE_CF_UNIQ (with PASTE_CF_KEYS): the arg stream holds one reference
 * per distinct resolution of the entry instead of one per binding --
 * bindings with the same expression (kind, path steps; fallback suffix,
 * start index and fail tool) on the same source event resolve to the same
 * node, so the plan numbers them as units in first-use order (map word bits
 * 56-63, the count in header byte 3) and the host maps each binding to its
 * unit's reference.
 * PASTE_CF_KEY8 (with PASTE_CF_KEYS): the key stream holds one u8 per
 * session instead of the u16 key: the entry's plan code, byte 8 of its
 * live-plan header, which the caller assigns after paste_build_live_plan
 * (one code per distinct non-empty entry content, 0xFF for every entry
 * without predictions or actions; the host maps a code back to a
 * representative key).  0xFF = no predictions.                           */
enum { PASTE_CF_HDR8 = 1, PASTE_CF_PRED8 = 2, PASTE_CF_ARG16 = 4, PASTE_CF_ENTRY16 = 8,
       PASTE_CF_KEYS = 16, PASTE_CF_UNIQ = 32, PASTE_CF_KEY8 = 64 };
typedef struct {
  void* hdr;         /* [n]                                                  */
  void* pred;
  void* arg;
  uint8_t* act;
  int64_t* totals;   /* [5]                                                  */
  int32_t format;    /* PASTE_CF_* bits                                       */
  int32_t pad;
} paste_compact_desc;

/* 1 when paste_predict_compact runs the fused kernel for this request shape
 * (else it returns PASTE_ERR_UNSUPPORTED and the caller runs
 * paste_predict_batch + paste_compact_records, which cannot produce
 * PASTE_CF_ENTRY16).  `pool` must carry its match table.                   */
int paste_predict_compact_supported(const paste_pool_desc* pool, int32_t window_capacity,
                                    int32_t max_candidates, int32_t max_bindings,
                                    int32_t format);

/* The serving step in one kernel: paste_predict_batch (observe + predict +
 * admit, same semantics) writing the step's records straight into the
 * narrow streams above instead of K fixed slots per session.  Needs the
 * match-table fast path (pool compiled with paste_build_match_table for
 * these max_candidates / window capacity), max_candidates <= 31 and
 * <= 16384 patterns; PASTE_ERR_UNSUPPORTED otherwise.  `scratch` is device
 * memory of paste_predict_compact_scratch_bytes(n_sessions) bytes.        */
int64_t paste_predict_compact_scratch_bytes(int64_t n_sessions);
int paste_predict_compact(const paste_pool_desc* pool, paste_windows* windows,
                          const paste_admit_desc* admit, int32_t max_candidates,
                          int32_t max_bindings, paste_compact_desc* out, void* scratch,
                          void* stream);
/* ---------------------------------------------------------------------- */
/* Live plan: the live step with its key-only work compiled (live_plan.cu)  */
/* ---------------------------------------------------------------------- */

/* Which patterns match, their rank order, the bindings to resolve and the
 * admit decisions (winner per tool, level if complete, utility) depend only
 * on the match-table key and the admit tables (policy.py:207-244: admission
 * does not depend on completeness, only the level does).  The plan holds
 * them per key; the walk table holds, per (binding, node), the node a
 * PathLookup / FormatTemplate binding resolves to in the tape starting at
 * that node (mappings.py:143-223; IndexedFallback is resolved at run time).
 * Rebuild the plan when the admit tables change (policy, EWMA estimates).  */
typedef struct {
  const void* plan;           /* paste_live_plan_bytes() bytes                */
  int32_t max_candidates;     /* K the plan was built for                     */
  int32_t max_bindings;       /* pool->max_bindings at build                  */
  const int32_t* walk;        /* [n_bindings][walk_nodes] or NULL             */
  int64_t walk_nodes;
} paste_live_plan;

/* -1 when outside the envelope: needs the pool's match table for (K, W),
 * K <= 31, gather depth <= 4, window capacity <= 16.                       */
int64_t paste_live_plan_bytes(const paste_pool_desc* pool, int32_t max_candidates,
                              int32_t window_capacity);
int paste_build_live_plan(const paste_pool_desc* pool, const paste_admit_desc* admit,
                          int32_t max_candidates, int32_t window_capacity, void* plan,
                          void* stream);
/* -1 above 2^24 entries.                                                    */
int64_t paste_live_walk_bytes(int32_t n_bindings, int64_t n_nodes);
int paste_build_live_walk(const paste_pool_desc* pool, int32_t n_bindings,
                          const paste_tape_node* nodes, int64_t n_nodes, int32_t* walk,
                          void* stream);

/* paste_predict_batch (observe + predict + admit, same records) from a live
 * plan: windows must observe (new_tok and new_ref / new_node set).          */
int paste_predict_live(const paste_pool_desc* pool, paste_windows* windows,
                       const paste_admit_desc* admit, const paste_live_plan* plan,
                       paste_predict_out* out, void* stream);
/* paste_predict_compact from a live plan (same streams and totals): the
 * pipelined step writes the fixed-position streams and an L2-resident
 * per-session staging record, then a scatter pass places the variable-length
 * streams (two launches).  scratch: device memory of
 * paste_predict_live_compact_scratch_bytes(n, K, max_bindings) bytes.     */
int64_t paste_predict_live_compact_scratch_bytes(int64_t n_sessions, int32_t max_candidates,
                                                 int32_t max_bindings);
int paste_predict_live_compact(const paste_pool_desc* pool, paste_windows* windows,
                               const paste_admit_desc* admit, const paste_live_plan* plan,
                               int32_t max_bindings, paste_compact_desc* out, void* scratch,
                               int64_t scratch_bytes, void* stream);

int64_t paste_compact_scratch_bytes(int64_t n_sessions);
int paste_compact_records(const paste_predict_out* out, int64_t n_sessions,
                          const paste_pool_desc* pool, paste_compact_desc* c, void* scratch,
                          void* stream);

/* ---------------------------------------------------------------------- */
/* K7: Phase II hypothesis hit counts (mappings.py:276-417, 326-335)        */
/* ---------------------------------------------------------------------- */

/* For every (hypothesis h, occurrence m): resolve hypothesis h's expression
 * against occurrence m's matched context and compare it with m's actual
 * argument (values_equal).  hits[h] / unsure[h] are accumulated (zero them
 * first); eq[h*n_occ + m] (optional) = 1 equal, 0 not, 2 unsure.  FormatTemplate
 * pairs involving non-ASCII text are "unsure" (the caller re-evaluates them
 * with Unicode string semantics).  fmt[5*h..] = prefix offset / length,
 * suffix offset / length (into fmt_bytes), normalization (0 none, 1 trim,
 * 2 lowercase).  occ_event / src_pos are [n_occ][n_ctx]; src_pos is the
 * matched event's first position in the occurrence's history (-1 absent),
 * history tokens of later copies of the same event are -1.                 */
typedef struct {
  int64_t n_hyp;
  int64_t n_occ;
  int32_t n_ctx;
  int32_t pad;
  const paste_binding* hyp;
  const int32_t* steps;
  const int32_t* fmt;
  const uint8_t* fmt_bytes;
  const paste_tape_node* nodes;
  const uint8_t* bytes;
  const paste_event_ref* refs;
  const int32_t* occ_event;
  const int32_t* src_pos;
  const int32_t* hist_off;   /* [n_occ + 1]                                   */
  const int32_t* hist_tok;
  const int32_t* act_type;   /* [n_occ] tape type of the actual argument      */
  const uint8_t* act_nan;    /* [n_occ]                                       */
  const int64_t* act_off;    /* [n_occ + 1] canonical bytes of the actual     */
  const uint8_t* act_bytes;
  int64_t* hits;             /* [n_hyp]                                       */
  int64_t* unsure;           /* [n_hyp]                                       */
  uint8_t* eq;               /* optional [n_hyp * n_occ]                      */
  /* corpus mode (mine() over one corpus tape): when
   * hist_end is set, occurrence m's history is hist_tok[hist_off[m],
   * hist_end[m]) -- overlapping ranges of the corpus token stream (bit 31 =
   * stream start) -- instead of the CSR hist_off[m], hist_off[m + 1]; when
   * act_event is set, the actual argument is node act_node[m] of tape
   * act_event[m] (-1: absent; containers never compare equal) instead of
   * act_type / act_nan / act_off / act_bytes.                               */
  const int32_t* hist_end;   /* optional [n_occ]                              */
  const int32_t* act_event;  /* optional [n_occ]                              */
  const int32_t* act_node;   /* [n_occ] with act_event                        */
} paste_holds_desc;

int paste_holds(const paste_holds_desc* d, void* stream);

/* Key lookup over many payload tapes: out_node[i] = the child of tape
 * tape[i]'s root dict whose key is `key` (node index inside the tape), -1
 * when the root is not a dict or has no such key; *n_scalar (device,
 * accumulated) += the number of found values that are scalars -- the
 * "present and not a container in every occurrence" test of
 * _common_scalar_args (mappings.py:299-315).                                */
typedef struct {
  int64_t n;
  const paste_tape_node* nodes;
  const paste_event_ref* refs;
  const int32_t* tape;
  int32_t key;
  int32_t pad;
  int32_t* out_node;
  uint64_t* n_scalar;
} paste_key_lookup_desc;

int paste_tape_key_lookup(const paste_key_lookup_desc* d, void* stream);

/* ---------------------------------------------------------------------- */
/* C2 replay: score_accuracy (prediction.py:133-169)                        */
/* ---------------------------------------------------------------------- */

/* Replays a trace corpus: every tool call after a session's first is
 * predicted from the window of the `call_len` events before it (the event
 * stream is all sessions back to back, LLM steps included as token -1), and
 * scored: top1 = first candidate's tool equals the call's tool, top3 = one of
 * the first three does, hit = some FULL candidate of that tool has canonical
 * arguments equal to the call's (canonical_arg_hash, events.py:117-118).
 * Arguments are compared by key set (key-set ids interned by the caller:
 * call_keyset / pat_keyset, -1 = "let the host decide", -2 = args are not a
 * dict) and per binding by canonical value: scalar type class + canonical
 * bytes (NFC for strings); FormatTemplate values compose prefix +
 * norm(leaf text) + suffix when everything is ASCII.  Calls whose outcome
 * needs Unicode or container semantics are flagged in `unsure` (the caller
 * re-checks them; their hit is not counted).  tallies = {top1, top3, hits,
 * unsure} (accumulated: zero them first).  cand_limit applies Python's
 * preds[:m] to each candidate list (INT32_MAX = no limit).  The prediction
 * records land in `out` (any layout) for the caller's re-check.  Windows are
 * read in place from the event stream (paste_windows stream mode).         */
enum { PASTE_FMT_NON_ASCII = 0x100 };
typedef struct {
  int64_t n_calls;
  int32_t capacity;          /* W = window_capacity                           */
  int32_t cand_limit;
  const int32_t* ev_tok;     /* [n_events] sig, -1 = LLM step                 */
  const int32_t* ev_evt;     /* [n_events] result payload index into refs     */
  const int64_t* call_pos;   /* [n_calls] stream index of the scored call     */
  const int64_t* call_len;   /* [n_calls] window length (<= W)                */
  const int32_t* call_tool;  /* [n_calls] tool id of the call                 */
  const int32_t* call_args;  /* [n_calls] args payload index into refs        */
  const int32_t* call_keyset;/* [n_calls]                                     */
  const int32_t* pat_keyset; /* [n_patterns]                                  */
  const int32_t* bind_key;   /* [n_bindings] key id of each binding's arg name*/
  const int32_t* fmt;        /* [5 * n_bindings] as paste_holds_desc.fmt, the
                                normalization word may carry
                                PASTE_FMT_NON_ASCII (prefix/suffix not ASCII) */
  const uint8_t* fmt_bytes;
  const paste_tape_node* nodes;
  const uint8_t* bytes;
  const paste_event_ref* refs;
  int64_t* tallies;          /* [4]                                           */
  uint8_t* unsure;           /* [n_calls]                                     */
} paste_replay_desc;

int paste_replay_score(const paste_pool_desc* pool, const paste_replay_desc* d,
                       paste_predict_out* out, void* stream);

/* The same replay as ONE kernel without prediction records (SURVEY 8(f)
 * row 3): per call the window's newest G tool events select a match-table
 * entry, top1 / top3 come from its records' tools, and only the FULL-
 * candidate-of-the-call's-tool bindings are resolved and compared.
 * tallies / unsure as paste_replay_score; the caller re-checks unsure calls
 * with paste_replay_score's records.  Requires pool->match_table valid for
 * max_candidates (mt_k >= max_candidates) with mt_g <= 8; else
 * PASTE_ERR_UNSUPPORTED.                                                   */
int paste_replay_fused(const paste_pool_desc* pool, const paste_replay_desc* d,
                       int32_t max_candidates, void* stream);

/* Number of kernel launches the last paste_* call on this thread issued.   */
int paste_last_launch_count(void);

/* n async copies (bytes[i] <= 0 skipped) on `stream`, in order.  Used by the
 * serving loop to issue a step's uploads / sized downloads in one call.    */
enum { PASTE_COPY_H2D = 1, PASTE_COPY_D2H = 2, PASTE_COPY_D2D = 3 };
int paste_memcpy_batch(int32_t n, void* const* dst, const void* const* src,
                       const int64_t* bytes, int32_t kind, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PASTE_H */
