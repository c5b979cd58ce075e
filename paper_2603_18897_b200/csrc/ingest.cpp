// Native columnar ingest of a JSONL trace for mining (host code, OpenMP).
//
// Reference: ingest_trace (events.py:196-252) with _parse_record (:165-184)
// and _split_on_gaps (:244-252): records are grouped by session_id in order
// of first appearance, each session is stably sorted by (t_start, seq)
// (a session whose seq order changed counts as reordered), split where
// t_start - previous t_end > threshold (over ALL events, LLM steps
// included), and mining reads each segment's tool events (Session.
// tool_events, events.py:66-72).  Output: the columnar trace of those tool
// events in segment order (session column = segment index), which the
// device count pass consumes with no further gap split.
//
// Lines are parsed in parallel.  A record with a missing required field is
// an ingest error (tallied by line number, as the reference does).  Anything
// whose Python semantics this parser does not reproduce exactly -- JSON it
// cannot validate, escapes in session / tool strings, non-string ids,
// non-integral or non-numeric seq, timestamps given as strings, NaN start
// times (unordered sort keys), duplicate keys, or text that str.splitlines()
// would split differently -- makes the call return PASTE_ERR_UNSUPPORTED so
// the caller runs the reference-semantics host ingest instead.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>
#include <algorithm>
#include <numeric>
#include <omp.h>
#include <memory>
#include <chrono>

#include "paste.h"

namespace paste {
void set_error(const char* fmt, ...);
void reset_launches();
}  // namespace paste

namespace {

// L_MISSING: a required field is absent; L_INVALID: Event.__post_init__
// rejects the record (events.py:59-63).  Both are tallied ingest errors.
enum LineKind : uint8_t { L_EMPTY, L_OK, L_MISSING, L_INVALID, L_ODD };

struct Rec {
  std::string_view session, tool;
  uint64_t sid_hash = 0, tool_hash = 0;  // computed in the parallel parse
  int64_t seq = 0;
  double t_start = 0, t_end = 0;
  int32_t line = 0;  // 1-based
  int32_t reason = 0;  // error code (paste_ingest_desc.error_codes)
  uint8_t kind = L_EMPTY;
  bool tool_call = true, success = true;
};

struct Cursor {
  const char* p;
  const char* e;
  bool ok = true;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool lit(const char* s) {
    const size_t n = strlen(s);
    if ((size_t)(e - p) < n || memcmp(p, s, n) != 0) return ok = false;
    p += n;
    return true;
  }
};

// JSON string (p at the opening quote); sets `escaped` when a backslash is
// seen; returns the raw body.  Control characters are rejected (json.loads
// strict mode).
std::string_view parse_string(Cursor& c, bool* escaped) {
  if (c.p >= c.e || *c.p != '"') { c.ok = false; return {}; }
  const char* b = ++c.p;
  *escaped = false;
  while (c.p < c.e) {
    const unsigned char ch = (unsigned char)*c.p;
    if (ch == '"') {
      std::string_view v(b, c.p - b);
      ++c.p;
      return v;
    }
    if (ch < 0x20) { c.ok = false; return {}; }
    if (ch == '\\') {
      *escaped = true;
      if (c.p + 1 >= c.e) { c.ok = false; return {}; }
      const char x = c.p[1];
      if (x == 'u') {
        if (c.e - c.p < 6) { c.ok = false; return {}; }
        for (int i = 2; i < 6; ++i)
          if (!isxdigit((unsigned char)c.p[i])) { c.ok = false; return {}; }
        c.p += 6;
        continue;
      }
      if (!strchr("\"\\/bfnrt", x)) { c.ok = false; return {}; }
      c.p += 2;
      continue;
    }
    ++c.p;
  }
  c.ok = false;
  return {};
}

// JSON number token (json.loads grammar plus NaN / Infinity / -Infinity);
// returns the token, sets `integral` for an int literal.
std::string_view parse_number(Cursor& c, bool* integral) {
  const char* b = c.p;
  *integral = true;
  if (c.p < c.e && *c.p == 'N') { *integral = false; c.lit("NaN"); return {b, size_t(c.p - b)}; }
  if (c.p < c.e && *c.p == '-') ++c.p;
  if (c.p < c.e && *c.p == 'I') { *integral = false; c.lit("Infinity"); return {b, size_t(c.p - b)}; }
  if (c.p >= c.e || !isdigit((unsigned char)*c.p)) { c.ok = false; return {}; }
  if (*c.p == '0') ++c.p;
  else while (c.p < c.e && isdigit((unsigned char)*c.p)) ++c.p;
  if (c.p < c.e && *c.p == '.') {
    *integral = false;
    ++c.p;
    if (c.p >= c.e || !isdigit((unsigned char)*c.p)) { c.ok = false; return {}; }
    while (c.p < c.e && isdigit((unsigned char)*c.p)) ++c.p;
  }
  if (c.p < c.e && (*c.p == 'e' || *c.p == 'E')) {
    *integral = false;
    ++c.p;
    if (c.p < c.e && (*c.p == '+' || *c.p == '-')) ++c.p;
    if (c.p >= c.e || !isdigit((unsigned char)*c.p)) { c.ok = false; return {}; }
    while (c.p < c.e && isdigit((unsigned char)*c.p)) ++c.p;
  }
  return {b, size_t(c.p - b)};
}

// skip any JSON value, validating it
void skip_value(Cursor& c, int depth) {
  c.ws();
  if (!c.ok || c.p >= c.e || depth > 512) { c.ok = false; return; }
  const char ch = *c.p;
  bool esc, integral;
  if (ch == '"') { parse_string(c, &esc); return; }
  if (ch == '{' || ch == '[') {
    const char close = ch == '{' ? '}' : ']';
    ++c.p;
    c.ws();
    if (c.p < c.e && *c.p == close) { ++c.p; return; }
    while (c.ok) {
      if (ch == '{') {
        c.ws();
        parse_string(c, &esc);
        c.ws();
        if (!c.ok || c.p >= c.e || *c.p != ':') { c.ok = false; return; }
        ++c.p;
      }
      skip_value(c, depth + 1);
      c.ws();
      if (!c.ok || c.p >= c.e) { c.ok = false; return; }
      if (*c.p == ',') { ++c.p; continue; }
      if (*c.p == close) { ++c.p; return; }
      c.ok = false;
    }
    return;
  }
  if (ch == 't') { c.lit("true"); return; }
  if (ch == 'f') { c.lit("false"); return; }
  if (ch == 'n') { c.lit("null"); return; }
  parse_number(c, &integral);
}

// ---------------------------------------------------------------------------
// payload tapes (tape.py layout) for _parse_record's args / result
// ---------------------------------------------------------------------------
struct TNode {
  uint8_t type, flags;
  uint16_t pad;
  int32_t key;
  uint32_t a, b;
};
static_assert(sizeof(TNode) == 16, "tape node is 16 bytes");

enum { T_NULL = 0, T_FALSE, T_TRUE, T_INT, T_FLOAT, T_STR, T_LIST, T_DICT };
enum { F_FLOATSRC = 2, F_NAN = 4, F_ASCII = 8 };

// Payload tapes land in per-thread arenas (no allocation per line); keys
// are interned per thread and renumbered globally after the parse.
struct Arena {
  std::vector<TNode> nodes;
  std::vector<uint8_t> bytes;
  std::unordered_map<std::string, int32_t> key_id;
  std::vector<const std::string*> key_name;  // id -> name (map nodes are stable)
  std::string scratch;
  int64_t byte_base = 0;  // byte offset of the tape being written
  int32_t intern(const std::string& k) {
    auto it = key_id.find(k);
    if (it != key_id.end()) return it->second;
    const int32_t id = (int32_t)key_name.size();
    it = key_id.emplace(k, id).first;
    key_name.push_back(&it->first);
    return id;
  }
};

// where one line's two tapes (result, args) live in its thread's arena
struct LineTapes {
  Arena* arena = nullptr;
  int64_t node0[2] = {0, 0}, nnode[2] = {0, 0}, byte0[2] = {0, 0}, nbyte[2] = {0, 0};
  bool has[2] = {false, false};
};

// Line starts and the str.splitlines() check, in parallel chunks.
bool split_lines(const char* text, int64_t len, std::vector<int64_t>& starts) {
  const int64_t CH = 1 << 22;
  const int64_t nch = (len + CH - 1) / CH;
  std::vector<std::vector<int64_t>> part(nch);
  bool odd = false;
#pragma omp parallel for schedule(static) reduction(|| : odd)
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t b = c * CH, e = std::min(len, b + CH);
    for (int64_t i = b; i < e; ++i) {
      const unsigned char ch = (unsigned char)text[i];
      if (ch == '\n') {
        if (i + 1 < len) part[c].push_back(i + 1);
      } else if (ch < 0x20 || ch >= 0xC2) {
        if (ch == '\r' || ch == '\v' || ch == '\f' || (ch >= 0x1c && ch <= 0x1e)) odd = true;
        else if (ch == 0xC2 && i + 1 < len && (unsigned char)text[i + 1] == 0x85) odd = true;
        else if (ch == 0xE2 && i + 2 < len && (unsigned char)text[i + 1] == 0x80 &&
                 ((unsigned char)text[i + 2] == 0xA8 || (unsigned char)text[i + 2] == 0xA9))
          odd = true;
      }
    }
  }
  starts.assign(1, 0);
  for (auto& p : part) starts.insert(starts.end(), p.begin(), p.end());
  return !odd;
}

void put_utf8(std::string& out, uint32_t cp) {
  if (cp < 0x80) {
    out += (char)cp;
  } else if (cp < 0x800) {
    out += (char)(0xC0 | (cp >> 6));
    out += (char)(0x80 | (cp & 0x3F));
  } else if (cp < 0x10000) {
    out += (char)(0xE0 | (cp >> 12));
    out += (char)(0x80 | ((cp >> 6) & 0x3F));
    out += (char)(0x80 | (cp & 0x3F));
  } else {
    out += (char)(0xF0 | (cp >> 18));
    out += (char)(0x80 | ((cp >> 12) & 0x3F));
    out += (char)(0x80 | ((cp >> 6) & 0x3F));
    out += (char)(0x80 | (cp & 0x3F));
  }
}

// JSON string -> UTF-8 text (json.loads).  `nfc_safe` is cleared when the
// text holds a lone surrogate or a code point >= U+0300 (its NFC form then
// needs the Unicode database: the caller hands the trace to the host);
// `ascii` tells whether every byte is < 0x80.
bool unescape(Cursor& c, std::string& out, bool* ascii, bool* nfc_safe) {
  bool esc;
  const std::string_view raw = parse_string(c, &esc);
  if (!c.ok) return false;
  out.clear();
  *ascii = true;
  *nfc_safe = true;
  for (size_t i = 0; i < raw.size();) {
    const unsigned char ch = (unsigned char)raw[i];
    if (ch == '\\') {
      const char x = raw[i + 1];
      if (x != 'u') {
        const char* m = "\"\\/bfnrt";
        const char* r = "\"\\/\b\f\n\r\t";
        out += r[strchr(m, x) - m];
        i += 2;
        continue;
      }
      uint32_t cp = (uint32_t)strtoul(std::string(raw.substr(i + 2, 4)).c_str(), nullptr, 16);
      i += 6;
      if (cp >= 0xD800 && cp < 0xDC00 && i + 6 <= raw.size() && raw[i] == '\\' &&
          raw[i + 1] == 'u') {
        const uint32_t lo =
            (uint32_t)strtoul(std::string(raw.substr(i + 2, 4)).c_str(), nullptr, 16);
        if (lo >= 0xDC00 && lo < 0xE000) {
          cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          i += 6;
        }
      }
      if (cp >= 0xD800 && cp < 0xE000) *nfc_safe = false;  // lone surrogate
      if (cp >= 0x80) *ascii = false;
      if (cp >= 0x300) *nfc_safe = false;
      put_utf8(out, cp);
      continue;
    }
    if (ch >= 0x80) {  // raw UTF-8 (valid: Python decoded the text)
      *ascii = false;
      uint32_t cp;
      int n;
      if (ch >= 0xF0) { cp = ch & 7; n = 3; }
      else if (ch >= 0xE0) { cp = ch & 15; n = 2; }
      else { cp = ch & 31; n = 1; }
      for (int k = 1; k <= n && i + k < raw.size(); ++k) cp = (cp << 6) | (raw[i + k] & 0x3F);
      if (cp >= 0x300) *nfc_safe = false;
      out.append(raw.data() + i, (size_t)n + 1);
      i += (size_t)n + 1;
      continue;
    }
    out += (char)ch;
    ++i;
  }
  return true;
}

// str(int(x)) of an integral double (exact, any magnitude)
std::string int_digits(double x) {
  const bool neg = x < 0;
  double ax = std::fabs(x);
  if (ax < 9.0e18) {
    const unsigned long long v = (unsigned long long)ax;
    std::string s = std::to_string(v);
    return (neg && v) ? "-" + s : s;
  }
  int e;
  const double f = std::frexp(ax, &e);                 // ax = f * 2^e, f in [0.5, 1)
  uint64_t m = (uint64_t)std::ldexp(f, 53);            // ax = m * 2^(e - 53)
  int shift = e - 53;
  std::vector<uint32_t> big;                           // base 1e9, little endian
  while (m) { big.push_back((uint32_t)(m % 1000000000ull)); m /= 1000000000ull; }
  while (shift > 0) {
    const int k = shift > 28 ? 28 : shift;
    uint64_t carry = 0;
    for (auto& d : big) {
      const uint64_t v = ((uint64_t)d << k) + carry;
      d = (uint32_t)(v % 1000000000ull);
      carry = v / 1000000000ull;
    }
    while (carry) { big.push_back((uint32_t)(carry % 1000000000ull)); carry /= 1000000000ull; }
    shift -= k;
  }
  std::string s = std::to_string(big.back());
  char buf[16];
  for (size_t i = big.size() - 1; i-- > 0;) {
    snprintf(buf, sizeof buf, "%09u", big[i]);
    s += buf;
  }
  return neg ? "-" + s : s;
}

// repr(x) of a finite non-integral double: the shortest digits that round
// trip (the correctly rounded p-digit form for the least p that does), in
// Python's float_repr_style layout (exponent when decpt <= -4 or > 16).
std::string py_repr(double x) {
  char buf[40];
  int p = 1;
  for (; p <= 17; ++p) {
    snprintf(buf, sizeof buf, "%.*e", p - 1, x);
    if (strtod(buf, nullptr) == x) break;
  }
  std::string t(buf);
  const bool neg = t[0] == '-';
  if (neg) t.erase(0, 1);
  const size_t epos = t.find('e');
  const int exp10 = atoi(t.c_str() + epos + 1);
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (t[i] != '.') digits += t[i];
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int decpt = exp10 + 1;
  std::string out;
  if (decpt <= -4 || decpt > 16) {
    out = digits.substr(0, 1);
    if (digits.size() > 1) out += "." + digits.substr(1);
    const int ex = decpt - 1;
    snprintf(buf, sizeof buf, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    out += buf;
  } else if (decpt <= 0) {
    out = "0." + std::string((size_t)-decpt, '0') + digits;
  } else if ((size_t)decpt >= digits.size()) {
    out = digits + std::string((size_t)decpt - digits.size(), '0') + ".0";
  } else {
    out = digits.substr(0, (size_t)decpt) + "." + digits.substr((size_t)decpt);
  }
  return neg ? "-" + out : out;
}

void push_scalar(Arena& t, int32_t key, uint8_t type, uint8_t flags, const char* data,
                 size_t len) {
  TNode nd{type, flags, 0, key, (uint32_t)((int64_t)t.bytes.size() - t.byte_base),
           (uint32_t)len};
  t.bytes.insert(t.bytes.end(), data, data + len);
  t.nodes.push_back(nd);
}

void push_scalar(Arena& t, int32_t key, uint8_t type, uint8_t flags, const std::string& v) {
  push_scalar(t, key, type, flags, v.data(), v.size());
}

// one JSON value -> tape nodes (pre-order; dict children in document order,
// which is json.loads' insertion order when no key repeats)
bool emit_value(Cursor& c, int32_t key, Arena& t, int depth) {
  c.ws();
  if (!c.ok || c.p >= c.e || depth > 512) return c.ok = false;
  const char ch = *c.p;
  if (ch == '{' || ch == '[') {
    const bool dict = ch == '{';
    const size_t idx = t.nodes.size();
    t.nodes.push_back(TNode{(uint8_t)(dict ? T_DICT : T_LIST), 0, 0, key, 0, 0});
    ++c.p;
    c.ws();
    uint32_t n = 0;
    int32_t seen_small[16];
    std::vector<int32_t> seen_big;
    if (c.p < c.e && *c.p == (dict ? '}' : ']')) {
      ++c.p;
    } else {
      while (true) {
        int32_t ck = -1;
        if (dict) {
          c.ws();
          bool ascii, safe;
          if (!unescape(c, t.scratch, &ascii, &safe) || !safe) return c.ok = false;
          ck = t.intern(t.scratch);
          // duplicate key (json.loads keeps the last value): host ingest
          for (uint32_t q = 0; q < n && q < 16; ++q)
            if (seen_small[q] == ck) return c.ok = false;
          if (n >= 16 && std::find(seen_big.begin(), seen_big.end(), ck) != seen_big.end())
            return c.ok = false;
          if (n < 16) seen_small[n] = ck;
          else seen_big.push_back(ck);
          c.ws();
          if (c.p >= c.e || *c.p != ':') return c.ok = false;
          ++c.p;
        }
        if (!emit_value(c, ck, t, depth + 1)) return false;
        ++n;
        c.ws();
        if (c.p < c.e && *c.p == ',') { ++c.p; continue; }
        if (c.p < c.e && *c.p == (dict ? '}' : ']')) { ++c.p; break; }
        return c.ok = false;
      }
    }
    t.nodes[idx].a = n;
    t.nodes[idx].b = (uint32_t)(t.nodes.size() - idx);
    return true;
  }
  if (ch == '"') {
    bool ascii, safe;
    if (!unescape(c, t.scratch, &ascii, &safe) || !safe) return c.ok = false;
    push_scalar(t, key, T_STR, ascii ? F_ASCII : 0, t.scratch);
    return true;
  }
  if (ch == 't') { if (!c.lit("true")) return false; push_scalar(t, key, T_TRUE, 0, "", 0); return true; }
  if (ch == 'f') { if (!c.lit("false")) return false; push_scalar(t, key, T_FALSE, 0, "", 0); return true; }
  if (ch == 'n') { if (!c.lit("null")) return false; push_scalar(t, key, T_NULL, 0, "", 0); return true; }
  bool integral;
  const std::string_view v = parse_number(c, &integral);
  if (!c.ok || v.empty()) return c.ok = false;
  if (integral) {  // int(literal): "-0" is 0
    if (v == "-0") push_scalar(t, key, T_INT, F_ASCII, "0", 1);
    else push_scalar(t, key, T_INT, F_ASCII, v.data(), v.size());
    return true;
  }
  double x;
  if (v == "NaN") x = NAN;
  else if (v == "Infinity") x = INFINITY;
  else if (v == "-Infinity") x = -INFINITY;
  else x = strtod(std::string(v).c_str(), nullptr);
  if (std::isnan(x)) push_scalar(t, key, T_FLOAT, F_NAN | F_ASCII, "nan", 3);
  else if (std::isinf(x)) push_scalar(t, key, T_FLOAT, F_ASCII, x > 0 ? "inf" : "-inf", x > 0 ? 3 : 4);
  else if (x == std::floor(x)) push_scalar(t, key, T_INT, F_FLOATSRC | F_ASCII, int_digits(x));
  else push_scalar(t, key, T_FLOAT, F_ASCII, py_repr(x));
  return true;
}

// One line -> record.  L_ODD = outside what this parser reproduces exactly.
// With `lt`, the record's `result` / `args` values become payload tapes.
void parse_line(const char* b, const char* e, Rec& r, LineTapes* lt = nullptr) {
  Cursor c{b, e};
  c.ws();
  if (c.p == c.e) { r.kind = L_EMPTY; return; }
  if (*c.p != '{') { r.kind = L_ODD; return; }
  ++c.p;
  enum { F_SESSION = 1, F_SEQ = 2, F_KIND = 4, F_TOOL = 8, F_STATUS = 16, F_TS = 32, F_TE = 64 };
  int seen = 0;
  c.ws();
  if (c.p < c.e && *c.p == '}') { ++c.p; }
  else while (true) {
    c.ws();
    bool esc;
    const std::string_view key = parse_string(c, &esc);
    c.ws();
    if (!c.ok || esc || c.p >= c.e || *c.p != ':') { r.kind = L_ODD; return; }
    ++c.p;
    c.ws();
    int field = 0;
    if (key == "session_id") field = F_SESSION;
    else if (key == "seq") field = F_SEQ;
    else if (key == "kind") field = F_KIND;
    else if (key == "tool") field = F_TOOL;
    else if (key == "status") field = F_STATUS;
    else if (key == "t_start_ms") field = F_TS;
    else if (key == "t_end_ms") field = F_TE;
    if (field & seen) { r.kind = L_ODD; return; }  // duplicate key: last wins in Python
    seen |= field;
    if (field == F_SESSION || field == F_TOOL || field == F_KIND || field == F_STATUS) {
      if (c.p >= c.e || *c.p != '"') { r.kind = L_ODD; return; }  // str(non-string)
      const std::string_view v = parse_string(c, &esc);
      if (!c.ok || esc) { r.kind = L_ODD; return; }
      if (field == F_SESSION) r.session = v;
      else if (field == F_TOOL) r.tool = v;
      else if (field == F_KIND) {
        if (v == "tool_call") r.tool_call = true;
        else if (v == "llm_step") r.tool_call = false;
        else { r.kind = L_ODD; return; }
      } else {
        if (v == "success") r.success = true;
        else if (v == "fail") r.success = false;
        else { r.kind = L_ODD; return; }
      }
    } else if (field == F_SEQ || field == F_TS || field == F_TE) {
      bool integral;
      const std::string_view v = parse_number(c, &integral);
      if (!c.ok || v.empty()) { r.kind = L_ODD; return; }
      const std::string tok(v);
      if (field == F_SEQ) {
        if (!integral || v.size() > 18) { r.kind = L_ODD; return; }
        r.seq = strtoll(tok.c_str(), nullptr, 10);
        if (r.seq < INT32_MIN || r.seq > INT32_MAX) { r.kind = L_ODD; return; }  // int32 column
      } else {
        double x;
        if (v == "NaN") x = NAN;
        else if (v == "Infinity") x = INFINITY;
        else if (v == "-Infinity") x = -INFINITY;
        else x = strtod(tok.c_str(), nullptr);  // correctly rounded, as Python's float()
        if (field == F_TS) {
          if (std::isnan(x)) { r.kind = L_ODD; return; }  // unordered sort key
          r.t_start = x;
        } else {
          r.t_end = x;
        }
      }
    } else if (lt && (key == "result" || key == "args")) {
      const int q = key == "result" ? 0 : 1;
      if (lt->has[q]) { r.kind = L_ODD; return; }  // duplicate field: last wins in Python
      lt->has[q] = true;
      Arena& a = *lt->arena;
      a.byte_base = (int64_t)a.bytes.size();
      lt->node0[q] = (int64_t)a.nodes.size();
      lt->byte0[q] = a.byte_base;
      if (!emit_value(c, -1, a, 1)) { r.kind = L_ODD; return; }
      lt->nnode[q] = (int64_t)a.nodes.size() - lt->node0[q];
      lt->nbyte[q] = (int64_t)a.bytes.size() - lt->byte0[q];
    } else {
      skip_value(c, 1);
      if (!c.ok) { r.kind = L_ODD; return; }
    }
    c.ws();
    if (c.p < c.e && *c.p == ',') { ++c.p; continue; }
    if (c.p < c.e && *c.p == '}') { ++c.p; break; }
    r.kind = L_ODD;
    return;
  }
  c.ws();
  if (c.p != c.e) { r.kind = L_ODD; return; }
  if (seen != 127) {
    r.kind = L_MISSING;
    r.reason = PASTE_INGEST_MISSING | (127 & ~seen);  // the absent fields, in _REQUIRED_FIELDS order
    return;
  }
  // Event.__post_init__ (events.py:59-63), in its order
  if (r.t_start > r.t_end) {
    r.kind = L_INVALID;
    r.reason = PASTE_INGEST_T_ORDER;
  } else if (r.tool_call && r.tool.empty()) {
    r.kind = L_INVALID;
    r.reason = PASTE_INGEST_EMPTY_TOOL;
  } else {
    r.kind = L_OK;
  }
}

// bytes that make str.splitlines() split where '\n' does not
bool odd_line_breaks(const char* t, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    const unsigned char c = (unsigned char)t[i];
    if (c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e)) return true;
    if (c == 0xC2 && i + 1 < n && (unsigned char)t[i + 1] == 0x85) return true;
    if (c == 0xE2 && i + 2 < n && (unsigned char)t[i + 1] == 0x80 &&
        ((unsigned char)t[i + 2] == 0xA8 || (unsigned char)t[i + 2] == 0xA9))
      return true;
  }
  return false;
}

}  // namespace

using paste::set_error;

extern "C" int paste_ingest_jsonl(const char* text, int64_t len, double inactivity_ms,
                                  paste_ingest_desc* d) {
  paste::reset_launches();
  if (!text || !d || len < 0) {
    set_error("null argument");
    return PASTE_ERR_INVALID;
  }
  if (odd_line_breaks(text, len)) {
    set_error("line separators other than '\\n': host ingest");
    return PASTE_ERR_UNSUPPORTED;
  }
  // line starts
  std::vector<int64_t> starts{0};
  for (int64_t i = 0; i < len; ++i)
    if (text[i] == '\n' && i + 1 < len) starts.push_back(i + 1);
  const int64_t n_lines = len == 0 ? 0 : (int64_t)starts.size();
  std::vector<Rec> recs(n_lines);
  bool odd = false;
#pragma omp parallel for schedule(dynamic, 4096) reduction(|| : odd)
  for (int64_t i = 0; i < n_lines; ++i) {
    const char* b = text + starts[i];
    const char* e = i + 1 < n_lines ? text + starts[i + 1] - 1 : text + len;
    if (e > b && e[-1] == '\n') --e;
    recs[i].line = (int32_t)(i + 1);
    parse_line(b, e, recs[i]);
    odd = odd || recs[i].kind == L_ODD;
  }
  if (odd) {
    set_error("records outside the native parser's exact subset: host ingest");
    return PASTE_ERR_UNSUPPORTED;
  }
  // sessions in first-appearance order; errors by line
  std::unordered_map<std::string_view, int32_t> sid;
  sid.reserve((size_t)n_lines / 4 + 16);
  std::vector<std::vector<int64_t>> members;
  std::vector<std::string_view> tools;
  std::unordered_map<std::string_view, int32_t> tool_id;
  int64_t n_err = 0;
  for (int64_t i = 0; i < n_lines; ++i) {
    const Rec& r = recs[i];
    if (r.kind == L_EMPTY) continue;
    if (r.kind == L_MISSING || r.kind == L_INVALID) {
      if (n_err < d->error_capacity) {
        if (d->error_lines) d->error_lines[n_err] = r.line;
        if (d->error_codes) {
          d->error_codes[n_err] = r.reason;
          if (d->error_seq) d->error_seq[n_err] = r.seq;
        }
      }
      ++n_err;
      continue;
    }
    auto it = sid.find(r.session);
    if (it == sid.end()) {
      it = sid.emplace(r.session, (int32_t)members.size()).first;
      members.emplace_back();
    }
    members[it->second].push_back(i);
    if (r.tool_call && !tool_id.count(r.tool)) {
      tool_id.emplace(r.tool, (int32_t)tools.size());
      tools.push_back(r.tool);
    }
  }
  // tools interned in sorted name order (sig order == (tool_type, status))
  std::vector<int32_t> order(tools.size());
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return tools[a] < tools[b]; });
  std::vector<int32_t> rank(tools.size());
  int64_t names_len = 0;
  for (size_t r = 0; r < order.size(); ++r) {
    rank[order[r]] = (int32_t)r;
    names_len += (int64_t)tools[order[r]].size() + 1;
  }
  if (d->tool_names && names_len <= d->tool_names_capacity) {
    char* w = d->tool_names;
    for (int32_t o : order) {
      memcpy(w, tools[o].data(), tools[o].size());
      w += tools[o].size();
      *w++ = '\0';
    }
  }
  d->n_tools = (int32_t)tools.size();
  d->tool_names_len = names_len;
  // per session: stable sort by (t_start, seq), gap split, tool events out
  int64_t n_out = 0, n_seg = 0, reordered = 0;
  for (auto& m : members) {
    std::vector<int64_t> sorted = m;
    std::stable_sort(sorted.begin(), sorted.end(), [&](int64_t a, int64_t b) {
      const Rec &x = recs[a], &y = recs[b];
      if (x.t_start != y.t_start) return x.t_start < y.t_start;
      return x.seq < y.seq;
    });
    bool changed = false;
    for (size_t k = 0; k < m.size(); ++k) changed |= recs[sorted[k]].seq != recs[m[k]].seq;
    reordered += changed;
    const Rec* prev = nullptr;
    for (int64_t i : sorted) {
      const Rec& r = recs[i];
      if (!prev || r.t_start - prev->t_end > inactivity_ms) ++n_seg;  // _split_on_gaps
      prev = &r;
      if (!r.tool_call) continue;
      if (n_out < d->capacity) {
        d->session[n_out] = (int32_t)(n_seg - 1);
        d->seq[n_out] = (int32_t)r.seq;
        d->t_start[n_out] = r.t_start;
        d->t_end[n_out] = r.t_end;
        d->sig[n_out] = 2 * rank[tool_id[r.tool]] + (r.success ? 1 : 0);
      }
      ++n_out;
    }
  }
  d->n_events = n_out;
  d->n_segments = n_seg;
  d->n_errors = n_err;
  d->n_lines = n_lines;
  d->reordered_sessions = reordered;
  if (n_out > d->capacity || (d->tool_names && names_len > d->tool_names_capacity)) {
    set_error("output capacity too small (need %lld events, %lld name bytes)",
              (long long)n_out, (long long)names_len);
    return PASTE_ERR_INVALID;
  }
  return PASTE_OK;
}


// ---------------------------------------------------------------------------
// raw parse for the device ingest path (paste_jsonl_*)
// ---------------------------------------------------------------------------
struct paste_jsonl {
  std::vector<int32_t> session, seq, sig, err_line, err_code;
  std::vector<int64_t> err_seq;
  std::vector<double> t_start, t_end;
  std::string tool_names, key_names;
  std::unique_ptr<TNode[]> nodes;  // default-initialised (no zero fill): written in parallel
  std::unique_ptr<uint8_t[]> bytes;
  std::unique_ptr<paste_event_ref[]> refs;
  int64_t n_nodes = 0, n_bytes = 0, n_refs = 0;
  int64_t n_sessions = 0, n_lines = 0, n_keys = 0;
  int32_t n_tools = 0;
};

namespace {
struct HashedView {  // a string view with its hash computed once
  std::string_view s;
  uint64_t h;
  bool operator==(const HashedView& o) const { return h == o.h && s == o.s; }
};
struct HashedViewHash {
  size_t operator()(const HashedView& v) const { return (size_t)v.h; }
};
}  // namespace

extern "C" int paste_jsonl_parse(const char* text, int64_t len, int32_t want_payloads,
                                 paste_jsonl** out) {
  paste::reset_launches();
  if (!text || !out || len < 0) {
    set_error("null argument");
    return PASTE_ERR_INVALID;
  }
  *out = nullptr;
  const bool prof = getenv("PASTE_JSONL_PROF") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t0 = now();
  auto lap = [&](const char* what) {
    if (!prof) return;
    const auto t1 = now();
    fprintf(stderr, "jsonl %-10s %.1f ms\n", what,
            std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  std::vector<int64_t> starts;
  if (!split_lines(text, len, starts)) {
    set_error("line separators other than '\\n': host ingest");
    return PASTE_ERR_UNSUPPORTED;
  }
  const int64_t n_lines = len == 0 ? 0 : (int64_t)starts.size();
  lap("split");
  std::vector<Rec> recs(n_lines);
  std::vector<LineTapes> tapes(want_payloads ? n_lines : 0);
  std::vector<std::unique_ptr<Arena>> arenas((size_t)omp_get_max_threads());
  for (auto& a : arenas) a.reset(new Arena());
  bool odd = false;
#pragma omp parallel for schedule(dynamic, 1024) reduction(|| : odd)
  for (int64_t i = 0; i < n_lines; ++i) {
    const char* b = text + starts[i];
    const char* e = i + 1 < n_lines ? text + starts[i + 1] - 1 : text + len;
    if (e > b && e[-1] == '\n') --e;
    recs[i].line = (int32_t)(i + 1);
    LineTapes* lt = nullptr;
    if (want_payloads) {
      lt = &tapes[i];
      lt->arena = arenas[(size_t)omp_get_thread_num()].get();
    }
    parse_line(b, e, recs[i], lt);
    if (recs[i].kind == L_OK) {
      recs[i].sid_hash = std::hash<std::string_view>()(recs[i].session);
      recs[i].tool_hash = std::hash<std::string_view>()(recs[i].tool);
    }
    odd = odd || recs[i].kind == L_ODD;
  }
  lap("parse");
  if (odd) {
    set_error("records outside the native parser's exact subset: host ingest");
    return PASTE_ERR_UNSUPPORTED;
  }
  auto* h = new paste_jsonl();
  h->n_lines = n_lines;
  // rows in file order: the ids need one sequential pass (first appearance),
  // everything else is filled in parallel afterwards
  std::unordered_map<HashedView, int32_t, HashedViewHash> sid, tool_id;
  sid.reserve((size_t)n_lines / 8 + 16);
  std::vector<std::string_view> tools;
  HashedView last_hv{}, last_tv{};
  int32_t last_sid = -1, last_tid = -1;
  std::vector<int64_t> row_line;  // line of every valid row
  std::vector<int32_t> row_sid, row_tid;
  row_line.reserve((size_t)n_lines);
  row_sid.reserve((size_t)n_lines);
  row_tid.reserve((size_t)n_lines);
  for (int64_t i = 0; i < n_lines; ++i) {
    const Rec& r = recs[i];
    if (r.kind == L_EMPTY) continue;
    if (r.kind == L_MISSING || r.kind == L_INVALID) {
      h->err_line.push_back(r.line);
      h->err_code.push_back(r.reason);
      h->err_seq.push_back(r.seq);
      continue;
    }
    const HashedView hv{r.session, r.sid_hash};
    if (!(last_sid >= 0 && hv == last_hv)) {  // records of a session mostly arrive together
      auto it = sid.find(hv);
      if (it == sid.end()) it = sid.emplace(hv, (int32_t)sid.size()).first;
      last_hv = hv;
      last_sid = it->second;
    }
    int32_t tid = -1;
    if (r.tool_call) {
      const HashedView tv{r.tool, r.tool_hash};
      if (!(last_tid >= 0 && tv == last_tv)) {
        auto t = tool_id.find(tv);
        if (t == tool_id.end()) {
          t = tool_id.emplace(tv, (int32_t)tools.size()).first;
          tools.push_back(r.tool);
        }
        last_tv = tv;
        last_tid = t->second;
      }
      tid = last_tid;
    }
    row_line.push_back(i);
    row_sid.push_back(last_sid);
    row_tid.push_back(tid);
  }
  {
    const int64_t nr = (int64_t)row_line.size();
    h->session.resize((size_t)nr);
    h->seq.resize((size_t)nr);
    h->sig.resize((size_t)nr);
    h->t_start.resize((size_t)nr);
    h->t_end.resize((size_t)nr);
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < nr; ++q) {
      const Rec& r = recs[row_line[q]];
      h->session[q] = row_sid[q];
      h->seq[q] = (int32_t)r.seq;
      h->t_start[q] = r.t_start;
      h->t_end[q] = r.t_end;
      const int32_t tid = row_tid[q];
      h->sig[q] = tid < 0 ? -1 : (tid << 1) | (r.success ? 1 : 0);  // tool rank applied below
    }
  }
  const int64_t n_rows = (int64_t)row_line.size();
  lap("rows");
  int64_t n_keys = 0;
  if (want_payloads) {
    // global key ids in sorted key order (deterministic), a remap per arena
    std::vector<std::string_view> all;
    for (auto& a : arenas)
      for (const std::string* k : a->key_name) all.push_back(*k);
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    std::unordered_map<std::string_view, int32_t> key_id;
    for (size_t k = 0; k < all.size(); ++k) {
      key_id.emplace(all[k], (int32_t)k);
      h->key_names.append(all[k].data(), all[k].size());
      h->key_names.push_back('\0');
    }
    n_keys = (int64_t)all.size();
    std::unordered_map<const Arena*, std::vector<int32_t>> remap;
    for (auto& a : arenas) {
      std::vector<int32_t>& rm = remap[a.get()];
      rm.resize(a->key_name.size());
      for (size_t k = 0; k < rm.size(); ++k) rm[k] = key_id.at(std::string_view(*a->key_name[k]));
    }
    // tape offsets (absent payload = one null node), then a parallel copy
    std::vector<int64_t> node_off(2 * n_rows + 1, 0), byte_off(2 * n_rows + 1, 0);
    for (int64_t r = 0; r < n_rows; ++r) {
      const LineTapes& lt = tapes[row_line[r]];
      for (int q = 0; q < 2; ++q) {
        const int64_t j = 2 * r + q;
        node_off[j + 1] = node_off[j] + (lt.nnode[q] ? lt.nnode[q] : 1);
        byte_off[j + 1] = byte_off[j] + lt.nbyte[q];
      }
    }
    h->n_nodes = node_off[2 * n_rows];
    h->n_bytes = byte_off[2 * n_rows];
    h->n_refs = 2 * n_rows;
    h->nodes.reset(new TNode[(size_t)h->n_nodes + 1]);
    h->bytes.reset(new uint8_t[(size_t)h->n_bytes + 1]);
    h->refs.reset(new paste_event_ref[(size_t)h->n_refs + 1]);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t r = 0; r < n_rows; ++r) {
      const LineTapes& lt = tapes[row_line[r]];
      const std::vector<int32_t>& rm = remap.at(lt.arena);
      for (int q = 0; q < 2; ++q) {
        const int64_t j = 2 * r + q;
        h->refs[(size_t)j] = paste_event_ref{node_off[j], byte_off[j]};
        TNode* dst = h->nodes.get() + node_off[j];
        if (lt.nnode[q] == 0) {
          *dst = TNode{T_NULL, 0, 0, -1, 0, 0};  // absent: record.get -> None
          continue;
        }
        const TNode* src = lt.arena->nodes.data() + lt.node0[q];
        for (int64_t x = 0; x < lt.nnode[q]; ++x) {
          TNode nd = src[x];
          if (nd.key >= 0) nd.key = rm[(size_t)nd.key];
          dst[x] = nd;
        }
        if (lt.nbyte[q])
          memcpy(h->bytes.get() + byte_off[j], lt.arena->bytes.data() + lt.byte0[q],
                 (size_t)lt.nbyte[q]);
      }
    }
  }
  lap("tapes");
  h->n_keys = n_keys;
  h->n_sessions = (int64_t)sid.size();
  // tools in sorted name order: sig = 2 * rank + success
  std::vector<int32_t> order(tools.size());
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return tools[a] < tools[b]; });
  std::vector<int32_t> rank(tools.size());
  for (size_t r = 0; r < order.size(); ++r) {
    rank[order[r]] = (int32_t)r;
    h->tool_names.append(tools[order[r]].data(), tools[order[r]].size());
    h->tool_names.push_back('\0');
  }
  for (auto& sg : h->sig)
    if (sg >= 0) sg = 2 * rank[sg >> 1] + (sg & 1);
  h->n_tools = (int32_t)tools.size();
  *out = h;
  return PASTE_OK;
}

extern "C" int paste_jsonl_sizes_of(const paste_jsonl* h, paste_jsonl_sizes* s) {
  if (!h || !s) {
    set_error("null argument");
    return PASTE_ERR_INVALID;
  }
  s->n_rows = (int64_t)h->session.size();
  s->n_sessions = h->n_sessions;
  s->n_errors = (int64_t)h->err_line.size();
  s->n_lines = h->n_lines;
  s->n_nodes = h->n_nodes;
  s->n_bytes = h->n_bytes;
  s->n_keys = h->n_keys;
  s->key_names_len = (int64_t)h->key_names.size();
  s->tool_names_len = (int64_t)h->tool_names.size();
  s->n_tools = h->n_tools;
  s->pad = 0;
  return PASTE_OK;
}

extern "C" int paste_jsonl_copy(const paste_jsonl* h, const paste_jsonl_out* o) {
  if (!h || !o) {
    set_error("null argument");
    return PASTE_ERR_INVALID;
  }
  auto cp = [](void* dst, const void* src, size_t n) {
    if (dst && n) memcpy(dst, src, n);
  };
  const size_t n = h->session.size();
  cp(o->session, h->session.data(), 4 * n);
  cp(o->seq, h->seq.data(), 4 * n);
  cp(o->t_start, h->t_start.data(), 8 * n);
  cp(o->t_end, h->t_end.data(), 8 * n);
  cp(o->sig, h->sig.data(), 4 * n);
  cp(o->error_lines, h->err_line.data(), 4 * h->err_line.size());
  cp(o->error_codes, h->err_code.data(), 4 * h->err_code.size());
  cp(o->error_seq, h->err_seq.data(), 8 * h->err_seq.size());
  cp(o->tool_names, h->tool_names.data(), h->tool_names.size());
  cp(o->nodes, h->nodes.get(), sizeof(TNode) * (size_t)h->n_nodes);
  cp(o->bytes, h->bytes.get(), (size_t)h->n_bytes);
  cp(o->refs, h->refs.get(), sizeof(paste_event_ref) * (size_t)h->n_refs);
  cp(o->key_names, h->key_names.data(), h->key_names.size());
  return PASTE_OK;
}

extern "C" void paste_jsonl_destroy(paste_jsonl* h) { delete h; }
