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

// One line -> record.  L_ODD = outside what this parser reproduces exactly.
void parse_line(const char* b, const char* e, Rec& r) {
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
