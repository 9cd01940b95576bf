// Fast `.klay` reader: the line-oriented text format of
// tensorize.py:197-313, parsed and validated in C++ so loading a 1M-node
// circuit takes a fraction of the Python parse. Accepts and rejects exactly
// what paper_2410_11415_b200/tensorized.py read_klay does (tests compare the
// two on round trips and on every rejection case); the structural checks are
// the rules of tensorize.py:94-132 (TensorizedCircuit.validate).
#include "klay.h"

#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

struct KlayFile {
  int64_t num_inputs = 0, num_vars = 0;
  std::vector<int64_t> roots;
  std::vector<int64_t> const_pos, const_val;
  std::vector<int64_t> lit_codes, lit_slots;
  std::vector<int64_t> widths, counts, sources, segments;
  std::vector<int8_t> ops;  // 0 product, 1 sum
};

namespace {

thread_local std::string g_file_err;

struct Fail {
  std::string msg;
};

constexpr int KLAY_FORMAT_VERSION = 1;

// one whitespace-separated line at a time, empty lines skipped
struct Lines {
  const char* p;
  const char* end;
  const char* b = nullptr;  // current line [b, e)
  const char* e = nullptr;
  static bool ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }
  bool next() {
    while (p < end) {
      const char* nl = static_cast<const char*>(memchr(p, '\n', (size_t)(end - p)));
      const char* le = nl ? nl : end;
      const char* q = p;
      p = nl ? nl + 1 : end;
      while (q < le && ws(*q)) ++q;
      if (q < le) {
        b = q;
        e = le;
        return true;
      }
    }
    return false;
  }
};

// tokens of one line
struct Toks {
  const char* p;
  const char* end;
  bool next(const char*& tb, const char*& te) {
    while (p < end && Lines::ws(*p)) ++p;
    if (p >= end) return false;
    tb = p;
    while (p < end && !Lines::ws(*p)) ++p;
    te = p;
    return true;
  }
};

std::string str(const char* b, const char* e) { return std::string(b, (size_t)(e - b)); }

// a decimal integer token (optional sign), as Python's int() on our writer's output
bool parse_i64(const char* b, const char* e, int64_t& v) {
  if (b >= e) return false;
  const char* q = b;
  bool neg = false;
  if (*q == '+' || *q == '-') {
    neg = *q == '-';
    ++q;
  }
  if (q >= e) return false;
  uint64_t acc = 0;
  for (; q < e; ++q) {
    if (*q < '0' || *q > '9') return false;
    const uint64_t d = (uint64_t)(*q - '0');
    if (acc > (UINT64_MAX - d) / 10) return false;
    acc = acc * 10 + d;
  }
  if (!neg && acc > (uint64_t)INT64_MAX) return false;
  if (neg && acc > (uint64_t)INT64_MAX + 1) return false;
  v = neg ? (int64_t)(0 - acc) : (int64_t)acc;
  return true;
}

int64_t need_i64(const char* b, const char* e) {
  int64_t v;
  if (!parse_i64(b, e, v)) throw Fail{"invalid integer " + str(b, e)};
  return v;
}

bool word_is(const char* b, const char* e, const char* w) {
  const size_t n = strlen(w);
  return (size_t)(e - b) == n && memcmp(b, w, n) == 0;
}

// the header word of the current line; returns the token cursor after it
Toks line_head(const Lines& ln, const char*& hb, const char*& he) {
  Toks t{ln.b, ln.e};
  t.next(hb, he);
  return t;
}

void expect_line(Lines& ln, const char* want, Toks& t) {
  if (!ln.next()) throw Fail{std::string("unexpected end of file, wanted '") + want + "'"};
  const char *hb, *he;
  t = line_head(ln, hb, he);
  if (!word_is(hb, he, want))
    throw Fail{std::string("expected '") + want + "' line, got '" + str(hb, he) + "'"};
}

// the integers after the header word (at most `limit` when >= 0)
void read_ints(Toks& t, std::vector<int64_t>& out) {
  const char *b, *e;
  while (t.next(b, e)) out.push_back(need_i64(b, e));
}

// "a:b" pair; b == nullptr slots reject a missing colon like partition()
void split_pair(const char* b, const char* e, const char*& m) {
  m = static_cast<const char*>(memchr(b, ':', (size_t)(e - b)));
}

void validate(const KlayFile& f) {
  // tensorize.py:94-132
  if (f.num_inputs < 0 || f.num_vars < 0) throw Fail{"negative input or variable count"};
  {
    std::vector<int64_t> s = f.lit_slots;
    std::sort(s.begin(), s.end());
    bool ok = (int64_t)s.size() == f.num_inputs;
    for (size_t i = 0; ok && i < s.size(); ++i) ok = s[i] == (int64_t)i;
    if (!ok) throw Fail{"input map does not cover slots 0..K-1 exactly once"};
  }
  for (int64_t code : f.lit_codes)
    if ((code < 0 ? -code : code) > f.num_vars)
      throw Fail{"input literal " + std::to_string(code) + " exceeds declared vars"};
  int64_t prev = f.num_inputs, e0 = 0;
  std::vector<char> seen;
  for (size_t l = 0; l < f.widths.size(); ++l) {
    const std::string where = "layer " + std::to_string(l + 1);
    const int8_t expected = (l % 2 == 0) ? 0 : 1;
    if (f.ops[l] != expected)
      throw Fail{where + " op '" + (f.ops[l] ? "sum" : "prod") + "', expected '" +
                 (expected ? "sum" : "prod") + "'"};
    const int64_t W = f.widths[l], E = f.counts[l];
    if (W <= 0) throw Fail{where + " has nonpositive width"};
    if (E == 0) throw Fail{where + " has no edges"};
    const int64_t* S = f.sources.data() + e0;
    const int64_t* R = f.segments.data() + e0;
    for (int64_t e = 1; e < E; ++e)
      if (R[e] < R[e - 1]) throw Fail{where + ": aggregation indices not nondecreasing"};
    bool cover = R[0] == 0 && R[E - 1] == W - 1;
    for (int64_t e = 1; cover && e < E; ++e) cover = R[e] - R[e - 1] <= 1;
    if (!cover) throw Fail{where + ": aggregation indices must cover 0..width-1"};
    seen.assign((size_t)std::max<int64_t>(prev, 0), 0);
    int64_t distinct = 0;
    for (int64_t e = 0; e < E; ++e) {
      if (S[e] < 0 || S[e] >= prev) throw Fail{where + ": edge index out of range"};
      if (!seen[(size_t)S[e]]) {
        seen[(size_t)S[e]] = 1;
        ++distinct;
      }
    }
    if (distinct != prev) throw Fail{where + ": some previous-layer node is never read"};
    prev = W;
    e0 += E;
  }
  for (int64_t r : f.roots)
    if (r < 0 || r >= prev) throw Fail{"root index " + std::to_string(r) + " outside final layer"};
  const int64_t num_roots = (int64_t)(f.roots.size() + f.const_pos.size());
  for (int64_t pos : f.const_pos)
    if (pos < 0 || pos >= num_roots) throw Fail{"constant root position out of range"};
}

void parse(const char* text, int64_t len, KlayFile& f) {
  Lines ln{text, text + len};
  Toks t{nullptr, nullptr};
  const char *b, *e;
  if (!ln.next()) throw Fail{"empty file"};
  {
    const char *hb, *he;
    t = line_head(ln, hb, he);
    if (!word_is(hb, he, "klay")) throw Fail{"expected 'klay' line, got '" + str(hb, he) + "'"};
    std::vector<int64_t> v;
    const char *vb, *ve;
    if (!t.next(vb, ve) || t.next(b, e)) throw Fail{"malformed version header"};
    for (const char* q = vb; q < ve; ++q)
      if (*q < '0' || *q > '9') throw Fail{"malformed version header"};
    if (need_i64(vb, ve) != KLAY_FORMAT_VERSION) throw Fail{"unsupported format version " + str(vb, ve)};
  }
  auto single = [&](const char* word, int64_t& out) {
    expect_line(ln, word, t);
    const char *vb, *ve;
    if (!t.next(vb, ve) || t.next(b, e)) throw Fail{std::string("malformed ") + word + " line"};
    out = need_i64(vb, ve);
  };
  single("inputs", f.num_inputs);
  single("vars", f.num_vars);
  expect_line(ln, "roots", t);
  read_ints(t, f.roots);
  bool have = ln.next();
  const char *hb = nullptr, *he = nullptr;
  if (have) t = line_head(ln, hb, he);
  if (have && word_is(hb, he, "constants")) {
    while (t.next(b, e)) {
      const char* m;
      split_pair(b, e, m);
      const char* vb = m ? m + 1 : e;
      if (!(e - vb == 1 && (*vb == '0' || *vb == '1')))
        throw Fail{"malformed constants entry '" + str(b, e) + "'"};
      const int64_t pos = need_i64(b, m);
      if (std::find(f.const_pos.begin(), f.const_pos.end(), pos) != f.const_pos.end())
        throw Fail{"duplicate constant root position " + std::to_string(pos)};
      f.const_pos.push_back(pos);
      f.const_val.push_back(*vb == '1' ? 1 : 0);
    }
    have = ln.next();
    if (have) t = line_head(ln, hb, he);
  }
  if (!have || !word_is(hb, he, "inputmap")) throw Fail{"missing inputmap line"};
  {
    std::vector<int64_t> codes;
    while (t.next(b, e)) {
      const char* m;
      split_pair(b, e, m);
      int64_t code = 0;
      if (!m || !parse_i64(b, m, code) || code == 0)
        throw Fail{"malformed inputmap entry '" + str(b, e) + "'"};
      f.lit_codes.push_back(code);
      f.lit_slots.push_back(need_i64(m + 1, e));
    }
    codes = f.lit_codes;
    std::sort(codes.begin(), codes.end());
    if (std::adjacent_find(codes.begin(), codes.end()) != codes.end())
      throw Fail{"duplicate literal in inputmap"};
  }
  while (ln.next()) {
    t = line_head(ln, hb, he);
    std::vector<const char*> tk;
    const char *xb, *xe;
    while (t.next(xb, xe)) {
      tk.push_back(xb);
      tk.push_back(xe);
    }
    if (!word_is(hb, he, "layer") || tk.size() != 8)
      throw Fail{"expected layer header, got '" + str(ln.b, ln.e) + "'"};
    const int64_t idx = need_i64(tk[0], tk[1]);
    const int64_t width = need_i64(tk[4], tk[5]);
    const int64_t ne = need_i64(tk[6], tk[7]);
    if (idx != (int64_t)f.widths.size() + 1) throw Fail{"layer " + std::to_string(idx) + " out of sequence"};
    int8_t op;
    if (word_is(tk[2], tk[3], "prod")) op = 0;
    else if (word_is(tk[2], tk[3], "sum")) op = 1;
    else throw Fail{"unknown layer op '" + str(tk[2], tk[3]) + "'"};
    const size_t s0 = f.sources.size(), r0 = f.segments.size();
    expect_line(ln, "S", t);
    read_ints(t, f.sources);
    expect_line(ln, "R", t);
    read_ints(t, f.segments);
    if ((int64_t)(f.sources.size() - s0) != ne || (int64_t)(f.segments.size() - r0) != ne)
      throw Fail{"layer " + std::to_string(idx) + ": edge count mismatch with header"};
    f.widths.push_back(width);
    f.counts.push_back(ne);
    f.ops.push_back(op);
  }
  validate(f);
}

}  // namespace

extern "C" int klay_read_klay(const char* text, int64_t len, KlayFile** out) {
  if (!out) return KLAY_EINVAL;
  *out = nullptr;
  if (!text && len > 0) return KLAY_EINVAL;
  KlayFile* f = new KlayFile();
  try {
    parse(text ? text : "", len, *f);
  } catch (const Fail& x) {
    g_file_err = x.msg;
    delete f;
    return KLAY_EFORMAT;
  } catch (...) {
    g_file_err = "out of memory";
    delete f;
    return KLAY_EINVAL;
  }
  *out = f;
  return KLAY_OK;
}

extern "C" const char* klay_read_klay_error(void) { return g_file_err.c_str(); }

extern "C" int klay_file_info(const KlayFile* f, int64_t* sizes) {
  if (!f || !sizes) return KLAY_EINVAL;
  sizes[0] = f->num_inputs;
  sizes[1] = f->num_vars;
  sizes[2] = (int64_t)f->widths.size();
  sizes[3] = (int64_t)f->sources.size();
  sizes[4] = (int64_t)f->roots.size();
  sizes[5] = (int64_t)f->const_pos.size();
  sizes[6] = (int64_t)f->lit_codes.size();
  return KLAY_OK;
}

extern "C" int klay_file_export(const KlayFile* f, int64_t* widths, int64_t* counts,
                                int64_t* sources, int64_t* segments, int64_t* roots,
                                int64_t* const_pos, int64_t* const_val, int64_t* lit_codes,
                                int64_t* lit_slots) {
  if (!f) return KLAY_EINVAL;
  auto put = [](const std::vector<int64_t>& v, int64_t* dst) {
    if (dst && !v.empty()) memcpy(dst, v.data(), v.size() * sizeof(int64_t));
  };
  put(f->widths, widths);
  put(f->counts, counts);
  put(f->sources, sources);
  put(f->segments, segments);
  put(f->roots, roots);
  put(f->const_pos, const_pos);
  put(f->const_val, const_val);
  put(f->lit_codes, lit_codes);
  put(f->lit_slots, lit_slots);
  return KLAY_OK;
}

extern "C" void klay_file_destroy(KlayFile* f) { delete f; }
