// io.cpp -- native readers / writers of the reference's file formats
// (reference io.py:33-182): DIMACS max-flow graphs, `u` update files and
// whitespace edge lists, feeding the GPU builder.  One buffered read of the
// file and a hand-rolled tokenizer; the accept / reject rules and the error
// texts are the reference's, line by line (io.py:20-31 ParseError, strip(),
// comment lines starting with 'c' or '#', str.split() fields, int() syntax).
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/mfx.h"

namespace mfx {
extern thread_local std::string g_last_error;
}

struct mfx_edges {
  int64_t n = 0, source = -1, sink = -1;
  std::vector<int64_t> us, vs, caps;
};

namespace {

thread_local int64_t g_line = 0;

int perr(int64_t line, const std::string &msg) {
  g_line = line;
  mfx::g_last_error = msg;
  return MFX_PARSE_ERROR;
}

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; }

// Python repr() of an ASCII line (the reference formats {line!r})
std::string py_repr(const std::string &s) {
  bool sq = s.find('\'') != std::string::npos, dq = s.find('"') != std::string::npos;
  char q = (sq && !dq) ? '"' : '\'';
  std::string out(1, q);
  for (unsigned char c : s) {
    if (c == (unsigned char)q || c == '\\') {
      out += '\\';
      out += (char)c;
    } else if (c == '\t') {
      out += "\\t";
    } else if (c == '\n') {
      out += "\\n";
    } else if (c == '\r') {
      out += "\\r";
    } else if (c < 0x20 || c == 0x7f) {
      char b[8];
      snprintf(b, sizeof(b), "\\x%02x", c);
      out += b;
    } else {
      out += (char)c;
    }
  }
  out += q;
  return out;
}

// Python int() of one whitespace-free token: optional sign, digits with
// single underscores between them.  false when int() would raise (or the
// value leaves int64, which the reference's int64 arrays cannot hold).
bool py_int(const char *p, size_t len, int64_t *out) {
  size_t i = 0;
  bool neg = false;
  if (i < len && (p[i] == '+' || p[i] == '-')) neg = p[i++] == '-';
  if (i >= len) return false;
  unsigned long long v = 0;
  bool digit_before = false;
  for (; i < len; ++i) {
    char c = p[i];
    if (c == '_') {
      if (!digit_before || i + 1 >= len || p[i + 1] < '0' || p[i + 1] > '9') return false;
      digit_before = false;
      continue;
    }
    if (c < '0' || c > '9') return false;
    if (v > (~0ull - 9) / 10) return false;
    v = v * 10 + (unsigned)(c - '0');
    digit_before = true;
  }
  if (!digit_before) return false;
  if (!neg && v > (unsigned long long)INT64_MAX) return false;
  if (neg && v > (unsigned long long)INT64_MAX + 1ull) return false;
  *out = neg ? (int64_t)(0 - v) : (int64_t)v;
  return true;
}

struct Line {
  std::string text;                // stripped line
  std::vector<std::string> parts;  // split fields
};

// Iterate the stripped, non-comment lines of a file.
struct Reader {
  std::vector<char> buf;
  size_t pos = 0;
  int64_t lineno = 0;
  bool open(const char *path) {
    FILE *f = fopen(path, "rb");
    if (!f) return false;
    char tmp[1 << 16];
    size_t r;
    while ((r = fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + r);
    fclose(f);
    return true;
  }
  // next non-comment line; false at EOF
  bool next(Line &ln) {
    while (pos < buf.size()) {
      size_t end = pos;
      while (end < buf.size() && buf[end] != '\n') ++end;
      size_t a = pos, b = end;
      pos = end < buf.size() ? end + 1 : end;
      ++lineno;
      while (a < b && is_space(buf[a])) ++a;
      while (b > a && is_space(buf[b - 1])) --b;
      if (a == b || buf[a] == 'c' || buf[a] == '#') continue;  // io.py:29-30
      ln.text.assign(&buf[a], b - a);
      ln.parts.clear();
      size_t i = a;
      while (i < b) {
        while (i < b && is_space(buf[i])) ++i;
        size_t j = i;
        while (j < b && !is_space(buf[j])) ++j;
        if (j > i) ln.parts.emplace_back(&buf[i], j - i);
        i = j;
      }
      return true;
    }
    return false;
  }
};

bool tok_int(const std::string &t, int64_t *v) { return py_int(t.data(), t.size(), v); }

}  // namespace

extern "C" {

int64_t mfx_io_error_line(void) { return g_line; }

// parse_graph (io.py:33-109)
int mfx_io_parse_graph(const char *path, mfx_edges **out) {
  *out = nullptr;
  Reader R;
  if (!R.open(path)) return perr(0, std::string("cannot open ") + path + ": " + strerror(errno));
  auto *E = new mfx_edges();
  bool have_p = false;
  int64_t n = 0, m = 0, arcs = 0, source = -1, sink = -1;
  Line ln;
  auto fail = [&](const std::string &msg) {
    delete E;
    return perr(R.lineno, msg);
  };
  while (R.next(ln)) {
    const std::string &kind = ln.parts[0];
    if (kind == "p") {
      if (have_p) return fail("duplicate problem line");
      if (ln.parts.size() != 4 || ln.parts[1] != "max")
        return fail("expected 'p max <n> <m>', got " + py_repr(ln.text));
      if (!tok_int(ln.parts[2], &n) || !tok_int(ln.parts[3], &m))
        return fail("bad problem line " + py_repr(ln.text));
      if (n <= 0 || m < 0)
        return fail("bad sizes n=" + std::to_string(n) + " m=" + std::to_string(m));
      have_p = true;
      E->us.resize((size_t)m);
      E->vs.resize((size_t)m);
      E->caps.resize((size_t)m);
    } else if (kind == "n") {
      if (!have_p) return fail("node line before problem line");
      if (ln.parts.size() != 3 || (ln.parts[2] != "s" && ln.parts[2] != "t"))
        return fail("expected 'n <id> s|t', got " + py_repr(ln.text));
      int64_t vid;
      if (!tok_int(ln.parts[1], &vid)) return fail("bad vertex id in " + py_repr(ln.text));
      if (vid < 1 || vid > n)
        return fail("vertex id " + std::to_string(vid) + " out of range [1, " + std::to_string(n) + "]");
      if (ln.parts[2] == "s") {
        if (source >= 0) return fail("duplicate source line");
        source = vid - 1;
      } else {
        if (sink >= 0) return fail("duplicate sink line");
        sink = vid - 1;
      }
    } else if (kind == "a") {
      if (!have_p) return fail("arc line before problem line");
      if (arcs >= m) return fail("more than " + std::to_string(m) + " arc lines");
      if (ln.parts.size() != 4) return fail("expected 'a <u> <v> <cap>', got " + py_repr(ln.text));
      int64_t u, v, c;
      if (!tok_int(ln.parts[1], &u) || !tok_int(ln.parts[2], &v) || !tok_int(ln.parts[3], &c))
        return fail("bad arc line " + py_repr(ln.text));
      if (u < 1 || u > n || v < 1 || v > n)
        return fail("arc endpoint out of range [1, " + std::to_string(n) + "] in " + py_repr(ln.text));
      if (c < 0) return fail("negative capacity in " + py_repr(ln.text));
      E->us[(size_t)arcs] = u - 1;
      E->vs[(size_t)arcs] = v - 1;
      E->caps[(size_t)arcs] = c;
      ++arcs;
    } else {
      return fail("unknown line kind " + py_repr(kind));
    }
  }
  R.lineno = 0;
  if (!have_p) return fail("missing problem line");
  if (source < 0) return fail("missing source node line");
  if (sink < 0) return fail("missing sink node line");
  if (arcs != m)
    return fail("header promised " + std::to_string(m) + " arcs, found " + std::to_string(arcs));
  E->n = n;
  E->source = source;
  E->sink = sink;
  *out = E;
  return MFX_OK;
}

// parse_updates (io.py:121-144), without the graph-side validation (the
// caller resolves the batch against the device graph)
int mfx_io_parse_updates(const char *path, int64_t n, mfx_edges **out) {
  *out = nullptr;
  Reader R;
  if (!R.open(path)) return perr(0, std::string("cannot open ") + path + ": " + strerror(errno));
  auto *E = new mfx_edges();
  Line ln;
  auto fail = [&](const std::string &msg) {
    delete E;
    return perr(R.lineno, msg);
  };
  while (R.next(ln)) {
    if (ln.parts[0] != "u" || ln.parts.size() != 4)
      return fail("expected 'u <from> <to> <new_cap>', got " + py_repr(ln.text));
    int64_t u, v, c;
    if (!tok_int(ln.parts[1], &u) || !tok_int(ln.parts[2], &v) || !tok_int(ln.parts[3], &c))
      return fail("bad update line " + py_repr(ln.text));
    if (u < 1 || u > n || v < 1 || v > n)
      return fail("vertex out of range [1, " + std::to_string(n) + "] in " + py_repr(ln.text));
    if (c < 0) return fail("negative capacity in " + py_repr(ln.text));
    E->us.push_back(u - 1);
    E->vs.push_back(v - 1);
    E->caps.push_back(c);
  }
  E->n = n;
  *out = E;
  return MFX_OK;
}

// parse_edge_list (io.py:153-182)
int mfx_io_parse_edge_list(const char *path, int one_indexed, mfx_edges **out) {
  *out = nullptr;
  Reader R;
  if (!R.open(path)) return perr(0, std::string("cannot open ") + path + ": " + strerror(errno));
  auto *E = new mfx_edges();
  Line ln;
  int64_t mx = -1;
  auto fail = [&](const std::string &msg) {
    delete E;
    return perr(R.lineno, msg);
  };
  while (R.next(ln)) {
    if (ln.parts.size() != 3) return fail("expected 'u v cap', got " + py_repr(ln.text));
    int64_t u, v, c;
    if (!tok_int(ln.parts[0], &u) || !tok_int(ln.parts[1], &v) || !tok_int(ln.parts[2], &c))
      return fail("bad edge line " + py_repr(ln.text));
    if (one_indexed) {
      u -= 1;
      v -= 1;
    }
    if (u < 0 || v < 0) return fail("negative vertex id in " + py_repr(ln.text));
    if (c < 0) return fail("negative capacity in " + py_repr(ln.text));
    E->us.push_back(u);
    E->vs.push_back(v);
    E->caps.push_back(c);
    mx = u > mx ? u : mx;
    mx = v > mx ? v : mx;
  }
  if (E->us.empty()) {
    R.lineno = 0;
    return fail("no edges found");
  }
  E->n = mx + 1;
  *out = E;
  return MFX_OK;
}

int mfx_edges_info(const mfx_edges *e, int64_t *info) {
  info[0] = e->n;
  info[1] = (int64_t)e->us.size();
  info[2] = e->source;
  info[3] = e->sink;
  return MFX_OK;
}

int mfx_edges_get(const mfx_edges *e, int64_t *us, int64_t *vs, int64_t *caps) {
  size_t m = e->us.size();
  if (m) {
    memcpy(us, e->us.data(), m * sizeof(int64_t));
    memcpy(vs, e->vs.data(), m * sizeof(int64_t));
    memcpy(caps, e->caps.data(), m * sizeof(int64_t));
  }
  return MFX_OK;
}

void mfx_edges_free(mfx_edges *e) { delete e; }

static int write_rows(FILE *f, const char *tag, int64_t m, const int64_t *us, const int64_t *vs,
                      const int64_t *caps) {
  std::string chunk;
  chunk.reserve(1 << 20);
  char b[96];
  for (int64_t i = 0; i < m; ++i) {
    int k = snprintf(b, sizeof(b), "%s %lld %lld %lld\n", tag, (long long)us[i] + 1,
                     (long long)vs[i] + 1, (long long)caps[i]);
    chunk.append(b, (size_t)k);
    if (chunk.size() > (1u << 20)) {
      if (fwrite(chunk.data(), 1, chunk.size(), f) != chunk.size()) return -1;
      chunk.clear();
    }
  }
  if (!chunk.empty() && fwrite(chunk.data(), 1, chunk.size(), f) != chunk.size()) return -1;
  return 0;
}

// write_graph (io.py:112-118)
int mfx_io_write_graph(const char *path, int64_t n, int64_t m, int64_t source, int64_t sink,
                       const int64_t *us, const int64_t *vs, const int64_t *caps) {
  FILE *f = fopen(path, "w");
  if (!f) return perr(0, std::string("cannot open ") + path + ": " + strerror(errno));
  fprintf(f, "p max %lld %lld\nn %lld s\nn %lld t\n", (long long)n, (long long)m,
          (long long)source + 1, (long long)sink + 1);
  int rc = write_rows(f, "a", m, us, vs, caps);
  if (fclose(f) != 0 || rc) return perr(0, std::string("write failed: ") + path);
  return MFX_OK;
}

// write_updates (io.py:147-150)
int mfx_io_write_updates(const char *path, int64_t k, const int64_t *us, const int64_t *vs,
                         const int64_t *caps) {
  FILE *f = fopen(path, "w");
  if (!f) return perr(0, std::string("cannot open ") + path + ": " + strerror(errno));
  int rc = write_rows(f, "u", k, us, vs, caps);
  if (fclose(f) != 0 || rc) return perr(0, std::string("write failed: ") + path);
  return MFX_OK;
}

}  // extern "C"
