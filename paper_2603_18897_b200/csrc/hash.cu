// canonical_arg_hash on the device: blake2b-128 of canonical_json(value).
//
// Reference (events.py:94-122):
//   canonical_form: dict keys NFC-normalised and sorted (by code point, which
//     is UTF-8 byte order), integral floats -> ints, strings NFC, lists kept;
//   canonical_json: json.dumps(..., sort_keys=True, separators=(",", ":"),
//     ensure_ascii=False);
//   canonical_arg_hash: hashlib.blake2b(text.encode("utf-8"), digest_size=16).
//
// One thread per value walks its payload tape depth-first (explicit stack),
// emits the canonical JSON bytes straight into a BLAKE2b block buffer and
// compresses every full block.  The tape already holds canonical scalar
// bytes (decimal for ints and integral floats, repr for other floats, NFC
// copies of strings), so the walk only adds JSON punctuation, string
// escaping (\" \\ \b \f \n \r \t, \u00XX for other control characters;
// everything else stays raw UTF-8) and NaN / Infinity spellings.  Dict
// children are emitted in key-rank order (ranks of the NFC key strings,
// computed once per key table on the host).  What the device cannot decide
// exactly is flagged "unsure" for the host: two keys of one dict with the
// same NFC form (canonical_form keeps the last), lone surrogates (the
// reference's .encode raises), nesting deeper than the stack, dicts wider
// than the rank scan bound.
#include "common.cuh"

namespace paste {

__constant__ uint64_t B2_IV[8] = {
    0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull, 0xa54ff53a5f1d36f1ull,
    0x510e527fade682d1ull, 0x9b05688c2b3e6c1full, 0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};

__constant__ uint8_t B2_SIGMA[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

__device__ __forceinline__ uint64_t rotr64(uint64_t x, int r) { return (x >> r) | (x << (64 - r)); }

#define B2_G(a, b, c, d, x, y)      \
  a = a + b + x;                    \
  d = rotr64(d ^ a, 32);            \
  c = c + d;                        \
  b = rotr64(b ^ c, 24);            \
  a = a + b + y;                    \
  d = rotr64(d ^ a, 16);            \
  c = c + d;                        \
  b = rotr64(b ^ c, 63);

struct Blake2b {
  uint64_t h[8];
  uint64_t t;        // bytes compressed so far
  uint8_t buf[128];  // pending block
  int fill;

  __device__ void init() {
    for (int i = 0; i < 8; ++i) h[i] = B2_IV[i];
    h[0] ^= 0x01010000ull ^ 16ull;  // digest 16 bytes, no key, fanout / depth 1
    t = 0;
    fill = 0;
  }
  __device__ void compress(bool last) {
    uint64_t m[16];
    for (int i = 0; i < 16; ++i) {
      uint64_t w = 0;
      for (int j = 7; j >= 0; --j) w = (w << 8) | buf[8 * i + j];
      m[i] = w;
    }
    uint64_t v[16];
    for (int i = 0; i < 8; ++i) {
      v[i] = h[i];
      v[i + 8] = B2_IV[i];
    }
    v[12] ^= t;  // byte counter (low word; payloads < 2^64 bytes)
    if (last) v[14] = ~v[14];
    for (int r = 0; r < 12; ++r) {
      const uint8_t* s = B2_SIGMA[r];
      B2_G(v[0], v[4], v[8], v[12], m[s[0]], m[s[1]]);
      B2_G(v[1], v[5], v[9], v[13], m[s[2]], m[s[3]]);
      B2_G(v[2], v[6], v[10], v[14], m[s[4]], m[s[5]]);
      B2_G(v[3], v[7], v[11], v[15], m[s[6]], m[s[7]]);
      B2_G(v[0], v[5], v[10], v[15], m[s[8]], m[s[9]]);
      B2_G(v[1], v[6], v[11], v[12], m[s[10]], m[s[11]]);
      B2_G(v[2], v[7], v[8], v[13], m[s[12]], m[s[13]]);
      B2_G(v[3], v[4], v[9], v[14], m[s[14]], m[s[15]]);
    }
    for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
  }
  // a full block is compressed only once more data arrives (the last block
  // is compressed by finish with the final flag)
  __device__ __forceinline__ void put(uint8_t c) {
    if (fill == 128) {
      t += 128;
      compress(false);
      fill = 0;
    }
    buf[fill++] = c;
  }
  __device__ void put_bytes(const uint8_t* p, int64_t n) {
    for (int64_t i = 0; i < n; ++i) put(p[i]);
  }
  __device__ void put_str(const char* s) {
    while (*s) put((uint8_t)*s++);
  }
  __device__ void finish(uint8_t* out16) {
    t += fill;
    for (int i = fill; i < 128; ++i) buf[i] = 0;
    compress(true);
    for (int i = 0; i < 16; ++i) out16[i] = (uint8_t)(h[i >> 3] >> (8 * (i & 7)));
  }
};

#undef B2_G

// JSON string body (ensure_ascii=False); false = lone surrogate (unsure)
__device__ bool put_json_string(Blake2b& b, const uint8_t* p, int64_t n) {
  const char* hex = "0123456789abcdef";
  b.put('"');
  for (int64_t i = 0; i < n; ++i) {
    const uint8_t c = p[i];
    if (c == 0xED && i + 1 < n && (p[i + 1] & 0xE0) == 0xA0) return false;  // U+D800..DFFF
    switch (c) {
      case '"': b.put('\\'); b.put('"'); break;
      case '\\': b.put('\\'); b.put('\\'); break;
      case '\n': b.put('\\'); b.put('n'); break;
      case '\r': b.put('\\'); b.put('r'); break;
      case '\t': b.put('\\'); b.put('t'); break;
      case '\b': b.put('\\'); b.put('b'); break;
      case '\f': b.put('\\'); b.put('f'); break;
      default:
        if (c < 0x20) {
          b.put('\\'); b.put('u'); b.put('0'); b.put('0');
          b.put((uint8_t)hex[c >> 4]); b.put((uint8_t)hex[c & 15]);
        } else {
          b.put(c);
        }
    }
  }
  b.put('"');
  return true;
}

constexpr int HSTACK = 32;        // container nesting handled on the device
constexpr int HDICT_SCAN = 256;   // widest dict ranked by the O(c^2) scan

struct HFrame {
  int32_t node;       // container node (relative to node_base)
  int32_t emitted;    // children written so far
  int32_t last_rank;  // dict: rank of the last child written
  int32_t cursor;     // list: next child node
};

__device__ __forceinline__ uint32_t node_size(const Node& n) { return n.size(); }

// canonical scalar bytes of a string node (NFC copy when flagged)
__device__ __forceinline__ const uint8_t* str_bytes(const uint8_t* bytes, int64_t byte_base,
                                                    const Node& nd, int64_t* len) {
  const uint8_t* p = bytes + byte_base + nd.a;
  if (nd.flags() & PASTE_F_NFC) {
    const uint8_t* q = p + nd.b;
    *len = (int64_t)q[0] | ((int64_t)q[1] << 8) | ((int64_t)q[2] << 16) | ((int64_t)q[3] << 24);
    return q + 4;
  }
  *len = nd.b;
  return p;
}

// emit a scalar node; false = unsure
__device__ bool put_scalar(Blake2b& b, const uint8_t* bytes, int64_t byte_base, const Node& nd) {
  switch (nd.type()) {
    case PASTE_T_NULL: b.put_str("null"); return true;
    case PASTE_T_TRUE: b.put_str("true"); return true;
    case PASTE_T_FALSE: b.put_str("false"); return true;
    case PASTE_T_INT: b.put_bytes(bytes + byte_base + nd.a, nd.b); return true;
    case PASTE_T_FLOAT: {
      const uint8_t* p = bytes + byte_base + nd.a;
      if (nd.flags() & PASTE_F_NAN) b.put_str("NaN");
      else if (nd.b == 3 && p[0] == 'i') b.put_str("Infinity");
      else if (nd.b == 4 && p[0] == '-' && p[1] == 'i') b.put_str("-Infinity");
      else b.put_bytes(p, nd.b);
      return true;
    }
    default: {
      int64_t len;
      const uint8_t* p = str_bytes(bytes, byte_base, nd, &len);
      return put_json_string(b, p, len);
    }
  }
}

struct KeyTab {  // NFC key strings and their code-point ranks (hashing.key_tables)
  const uint8_t* bytes;
  const int64_t* off;
  const int32_t* rank;
};

// Emit canonical_json of the tape value rooted at `root` (nodes relative to
// the event's node base); false = unsure (left to the host).
__device__ bool emit_tape_value(Blake2b& b, const paste_tape_node* nodes, const uint8_t* bytes,
                                int64_t bb, int32_t root, const KeyTab& K) {
  bool ok = true;
  HFrame st[HSTACK];
  int sp = 0;
  int32_t cur = root;  // node to emit next (-1: none, continue the top frame)
  bool first = true;   // inside the top frame: no separator before the next child
  while (ok) {
    if (cur >= 0) {
      const Node nd = load_node(nodes, cur);
      if (nd.type() < PASTE_T_LIST) {
        ok = put_scalar(b, bytes, bb, nd);
        cur = -1;
      } else {
        if (sp == HSTACK || (nd.type() == PASTE_T_DICT && nd.a > HDICT_SCAN)) return false;
        b.put(nd.type() == PASTE_T_DICT ? '{' : '[');
        st[sp++] = HFrame{cur, 0, -1, cur + 1};
        cur = -1;
        first = true;
        continue;
      }
    }
    if (sp == 0) break;  // the root is done
    // next child of the top frame
    HFrame& f = st[sp - 1];
    const Node fn = load_node(nodes, f.node);
    if (f.emitted == (int32_t)fn.a) {
      b.put(fn.type() == PASTE_T_DICT ? '}' : ']');
      --sp;
      first = false;
      continue;
    }
    if (!first) b.put(',');
    first = false;
    if (fn.type() == PASTE_T_LIST) {
      cur = f.cursor;
      f.cursor += (int32_t)node_size(load_node(nodes, cur));
      ++f.emitted;
      continue;
    }
    // dict: the child with the smallest key rank above the last one written
    int32_t best = -1, best_rank = 0x7fffffff, child = f.node + 1;
    bool tie = false;
    for (uint32_t c = 0; c < fn.a; ++c) {
      const Node cn = load_node(nodes, child);
      const int32_t r = K.rank[cn.key];
      if (r > f.last_rank) {
        if (r < best_rank) {
          best_rank = r;
          best = child;
          tie = false;
        } else if (r == best_rank) {
          tie = true;  // two keys with one NFC form: canonical_form keeps the last
        }
      }
      child += (int32_t)node_size(cn);
    }
    if (best < 0 || tie) return false;
    const Node kn = load_node(nodes, best);
    ok = put_json_string(b, K.bytes + K.off[kn.key], K.off[kn.key + 1] - K.off[kn.key]);
    b.put(':');
    f.last_rank = best_rank;
    ++f.emitted;
    cur = best;
  }
  return ok;
}

__global__ void canonical_hash_kernel(const paste_hash_desc D) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= D.n) return;
  const int64_t nb = D.refs[q].node_base, bb = D.refs[q].byte_base;
  Blake2b b;
  b.init();
  const bool ok = emit_tape_value(b, D.nodes + nb, D.bytes, bb, 0,
                                  KeyTab{D.key_bytes, D.key_off, D.key_rank});
  uint8_t* out = D.digest + 16 * q;
  if (ok) {
    b.finish(out);
  } else {
    for (int i = 0; i < 16; ++i) out[i] = 0;
  }
  D.unsure[q] = ok ? 0 : 1;
}

// ---------------------------------------------------------------------------
// Scheduler cache keys of admitted speculative actions (scheduling.py:464-480:
// key = (tool, canonical_arg_hash(prediction.args)) for every non-WARM_ONLY
// action).  A non-warm action's prediction is FULL, so every binding
// resolved: args = {arg_name: value} with value the resolved payload node
// (PathLookup / IndexedFallback) or prefix + norm(leaf_str(leaf)) + suffix
// (FormatTemplate, mappings.py:197-223).  One thread per session.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool py_space_c(uint8_t c) {  // str.isspace() on ASCII
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 28 && c <= 31);
}

// FormatTemplate value as a JSON string; false = unsure (non-ASCII text:
// Unicode strip / lower / NFC of the composed string are the host's)
__device__ bool emit_format(Blake2b& b, const paste_action_keys_desc& D, int bind,
                            const uint8_t* bytes, int64_t bb, const Node& leaf) {
  const int* f = D.fmt + 5 * bind;
  if (f[4] & PASTE_FMT_NON_ASCII) return false;
  const uint8_t* tb = bytes + bb + leaf.a;  // leaf_str: raw text / number text
  int64_t lo = 0, hi = leaf.b;
  for (int64_t i = lo; i < hi; ++i)
    if (tb[i] & 0x80) return false;
  const int norm = f[4] & 0xff;
  if (norm == 1) {  // str.strip()
    while (lo < hi && py_space_c(tb[lo])) ++lo;
    while (hi > lo && py_space_c(tb[hi - 1])) --hi;
  }
  const char* hex = "0123456789abcdef";
  auto esc = [&](uint8_t c) {
    switch (c) {
      case '"': b.put('\\'); b.put('"'); break;
      case '\\': b.put('\\'); b.put('\\'); break;
      case '\n': b.put('\\'); b.put('n'); break;
      case '\r': b.put('\\'); b.put('r'); break;
      case '\t': b.put('\\'); b.put('t'); break;
      case '\b': b.put('\\'); b.put('b'); break;
      case '\f': b.put('\\'); b.put('f'); break;
      default:
        if (c < 0x20) {
          b.put('\\'); b.put('u'); b.put('0'); b.put('0');
          b.put((uint8_t)hex[c >> 4]); b.put((uint8_t)hex[c & 15]);
        } else {
          b.put(c);
        }
    }
  };
  b.put('"');
  for (int i = 0; i < f[1]; ++i) esc(D.fmt_bytes[f[0] + i]);
  for (int64_t i = lo; i < hi; ++i) {
    uint8_t c = tb[i];
    if (norm == 2 && c >= 'A' && c <= 'Z') c += 32;  // str.lower() on ASCII
    esc(c);
  }
  for (int i = 0; i < f[3]; ++i) esc(D.fmt_bytes[f[2] + i]);
  b.put('"');
  return true;
}

__global__ void action_keys_kernel(const paste_action_keys_desc D) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = D.n_sessions;
  if (s >= n) return;
  const paste_predict_out& O = D.out;
  const KeyTab KT{D.key_bytes, D.key_off, D.key_rank};
  const int na = O.n_act[s];
  for (int j = 0; j < na; ++j) {
    const int64_t oj = out_at(O, n, s, j);
    uint8_t* key = D.keys + 16 * oj;
    if (O.act_level[oj] == 1) {  // WARM_ONLY: the scheduler's synthetic key
      D.key_state[oj] = 1;
      continue;
    }
    const int i = O.act_pred[oj];
    const int64_t oi = out_at(O, n, s, i);
    const paste_pattern pt = D.pool.patterns[O.pred_pat[oi]];
    const int nb = (pt.flags & PASTE_PF_HAS_MAPPING) ? pt.n_bind : 0;
    Blake2b b;
    b.init();
    b.put('{');
    bool ok = O.pred_comp[oi] == PASTE_C_FULL;
    int last = -1;
    for (int k = 0; ok && k < nb; ++k) {
      // bindings in the code-point order of their NFC arg names
      int best = -1, best_rank = 0x7fffffff;
      for (int bi = 0; bi < nb; ++bi) {
        const int r = KT.rank[D.bind_key[pt.bind_off + bi]];
        if (r > last && r < best_rank) {
          best_rank = r;
          best = bi;
        } else if (r == best_rank) {
          ok = false;  // two arg names with one NFC form
        }
      }
      if (best < 0) {
        ok = false;
        break;
      }
      last = best_rank;
      const int bind = pt.bind_off + best;
      const int key_id = D.bind_key[bind];
      if (k) b.put(',');
      ok = ok && put_json_string(b, KT.bytes + KT.off[key_id], KT.off[key_id + 1] - KT.off[key_id]);
      b.put(':');
      const int64_t ref = O.pred_arg[arg_at(O, n, s, i, best)];
      if (ref < 0) {
        ok = false;
        break;
      }
      const paste_event_ref er = D.refs[ref >> 32];
      const int32_t node = (int32_t)(ref & 0xffffffff);
      if (D.pool.bindings[bind].kind == PASTE_X_FORMAT)
        ok = ok && emit_format(b, D, bind, D.bytes, er.byte_base, load_node(D.nodes + er.node_base, node));
      else
        ok = ok && emit_tape_value(b, D.nodes + er.node_base, D.bytes, er.byte_base, node, KT);
    }
    b.put('}');
    if (ok) {
      b.finish(key);
      D.key_state[oj] = 0;
    } else {
      for (int t = 0; t < 16; ++t) key[t] = 0;
      D.key_state[oj] = 2;
    }
  }
}

}  // namespace paste

using namespace paste;

extern "C" int paste_canonical_hash(const paste_hash_desc* d, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null descriptor");
  if (d->n == 0) return PASTE_OK;
  PASTE_REQUIRE(d->nodes && d->bytes && d->refs && d->digest && d->unsure, "null array");
  const int threads = 128;
  canonical_hash_kernel<<<(unsigned)((d->n + threads - 1) / threads), threads, 0,
                          (cudaStream_t)stream>>>(*d);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}

extern "C" int paste_action_keys(const paste_action_keys_desc* d, void* stream) {
  reset_launches();
  PASTE_REQUIRE(d != nullptr, "null descriptor");
  if (d->n_sessions == 0) return PASTE_OK;
  PASTE_REQUIRE(d->out.n_act && d->out.act_pred && d->out.act_level && d->keys && d->key_state,
                "action records and key outputs are required");
  const int threads = 128;
  action_keys_kernel<<<(unsigned)((d->n_sessions + threads - 1) / threads), threads, 0,
                       (cudaStream_t)stream>>>(*d);
  count_launch();
  PASTE_CUDA_CHECK(cudaGetLastError());
  return PASTE_OK;
}
