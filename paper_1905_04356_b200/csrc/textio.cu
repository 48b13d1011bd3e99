// textio.cu -- interchange formats of dense polynomial matrices (host code).
//
// Text: the reference's CLI format, polmat_to_text / polmat_from_text
// (ref polmat.py:617-647): header "p m n", then one line per entry in
// row-major order, the trimmed coefficients low degree first separated by one
// space (the zero polynomial is an empty line), final newline.  Reading
// follows the reference exactly: lines as str.splitlines() cuts them, tokens
// as str.split() (Python whitespace), each token an integer of any size
// (sign, digits, '_' between digits) reduced with Python's `% p`, missing
// lines are zero entries, extra lines are ignored, ValueError on an empty
// text or a header that is not three integers.
//
// Binary (.fpmb, this library's own): little-endian header
//   "FPMB" u32 version=1 | u64 p | u32 m | u32 n | u32 L | u32 elem_bytes
// then m*n u32 trimmed lengths, then the dense m*n*L coefficients.  The
// Python side reads it with numpy (memmap-able, no parsing).
//
// Formatting and parsing run on all host threads (entries are independent:
// per-entry sizes, a prefix sum, then parallel writes).
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fpmat_b200.h"
#include "common.cuh"

namespace fpm {
namespace {

int nthreads() {
  unsigned h = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(h, 32u));
}

template <typename F>
void parallel_for(long long n, F f) {
  const int T = n < 4096 ? 1 : nthreads();
  if (T == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    const long long a = n * t / T, b = n * (t + 1) / T;
    th.emplace_back([=] { f(a, b); });
  }
  for (auto& x : th) x.join();
}

inline uint64_t elem(const void* M, int eb, size_t i) {
  return eb == 4 ? ((const uint32_t*)M)[i] : ((const uint64_t*)M)[i];
}

int trimmed(const void* M, int eb, size_t base, int L) {
  while (L > 0 && elem(M, eb, base + L - 1) == 0) --L;
  return L;
}

inline int digits(uint64_t v) {
  int d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

inline char* put_u64(char* o, uint64_t v) {
  char tmp[24];
  int k = 0;
  do {
    tmp[k++] = (char)('0' + v % 10);
    v /= 10;
  } while (v);
  while (k) *o++ = tmp[--k];
  return o;
}

// str.splitlines() boundaries for ASCII text: \n, \r, \r\n, \v, \f, \x1c-\x1e
inline bool line_break(unsigned char c) {
  return c == '\n' || c == '\r' || c == 0x0b || c == 0x0c || (c >= 0x1c && c <= 0x1e);
}
// str.split() whitespace for ASCII text
inline bool py_space(unsigned char c) {
  return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f);
}

struct Line {
  size_t a, b;  // [a, b)
};

std::vector<Line> split_lines(const char* t, size_t n) {
  std::vector<Line> out;
  size_t a = 0, i = 0;
  while (i < n) {
    const unsigned char c = (unsigned char)t[i];
    if (line_break(c)) {
      out.push_back({a, i});
      i += (c == '\r' && i + 1 < n && t[i + 1] == '\n') ? 2 : 1;
      a = i;
    } else {
      ++i;
    }
  }
  if (a < n) out.push_back({a, n});
  return out;
}

// Python int(token) % p; false if the token is not an integer literal
bool parse_mod(const char* s, size_t n, uint64_t p, uint64_t* out) {
  size_t i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) {
    neg = s[i] == '-';
    ++i;
  }
  if (i >= n) return false;
  u128 v = 0;
  bool prev_digit = false, any = false;
  for (; i < n; ++i) {
    const char c = s[i];
    if (c >= '0' && c <= '9') {
      v = (v * 10 + (unsigned)(c - '0')) % p;
      prev_digit = any = true;
    } else if (c == '_' && prev_digit && i + 1 < n && s[i + 1] >= '0' && s[i + 1] <= '9') {
      prev_digit = false;
    } else {
      return false;
    }
  }
  if (!any) return false;
  uint64_t r = (uint64_t)v;
  if (neg && r) r = p - r;
  *out = r;
  return true;
}

// tokens of one line
template <typename F>
bool for_tokens(const char* t, Line ln, F f) {
  size_t i = ln.a;
  while (i < ln.b) {
    while (i < ln.b && py_space((unsigned char)t[i])) ++i;
    if (i >= ln.b) break;
    size_t j = i;
    while (j < ln.b && !py_space((unsigned char)t[j])) ++j;
    if (!f(t + i, j - i)) return false;
    i = j;
  }
  return true;
}

bool parse_i64(const char* s, size_t n, long long* out) {
  size_t i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) {
    neg = s[i] == '-';
    ++i;
  }
  if (i >= n) return false;
  long long v = 0;
  for (; i < n; ++i) {
    if (s[i] == '_' && i > 0 && i + 1 < n) continue;
    if (s[i] < '0' || s[i] > '9') return false;
    if (v > (LLONG_MAX - 9) / 10) return false;
    v = v * 10 + (s[i] - '0');
  }
  *out = neg ? -v : v;
  return true;
}

int header(const char* t, const std::vector<Line>& lines, long long* p, long long* m,
           long long* n) {
  if (lines.empty()) {
    set_last_error("empty matrix file");
    return kInvalidArgument;
  }
  long long v[3];
  int cnt = 0;
  bool ok = for_tokens(t, lines[0], [&](const char* s, size_t len) {
    if (cnt >= 3) {
      ++cnt;
      return true;
    }
    if (!parse_i64(s, len, &v[cnt])) return false;
    ++cnt;
    return true;
  });
  if (!ok || cnt != 3) {
    set_last_error("matrix header must be 'p m n'");
    return kInvalidArgument;
  }
  *p = v[0];
  *m = v[1];
  *n = v[2];
  return kOk;
}

}  // namespace
}  // namespace fpm

using namespace fpm;

extern "C" {

int fpm_polmat_text_size(uint64_t p, int elem_bytes, const void* M, int m, int n, int L,
                         size_t* bytes) {
  if ((elem_bytes != 4 && elem_bytes != 8) || m < 0 || n < 0 || L < 0 || !bytes ||
      (!M && (long long)m * n * L > 0))
    return kInvalidArgument;
  const long long E = (long long)m * n;
  std::vector<size_t> sz((size_t)E);
  parallel_for(E, [&](long long a, long long b) {
    for (long long e = a; e < b; ++e) {
      const size_t base = (size_t)e * L;
      const int l = trimmed(M, elem_bytes, base, L);
      size_t s = 1;  // newline
      for (int t = 0; t < l; ++t) s += digits(elem(M, elem_bytes, base + t)) + (t ? 1 : 0);
      sz[e] = s;
    }
  });
  size_t tot = std::to_string(p).size() + std::to_string(m).size() + std::to_string(n).size() + 3;
  for (auto s : sz) tot += s;
  *bytes = tot;
  return kOk;
}

// polmat_to_text of a dense host matrix (polmat.py:617-623); out must hold
// fpm_polmat_text_size bytes (no terminating NUL is written)
int fpm_polmat_to_text(uint64_t p, int elem_bytes, const void* M, int m, int n, int L, char* out,
                       size_t cap, size_t* written) {
  if ((elem_bytes != 4 && elem_bytes != 8) || m < 0 || n < 0 || L < 0 || !out)
    return kInvalidArgument;
  const long long E = (long long)m * n;
  std::vector<size_t> off((size_t)E + 1, 0);
  const std::string head = std::to_string(p) + " " + std::to_string(m) + " " + std::to_string(n) + "\n";
  parallel_for(E, [&](long long a, long long b) {
    for (long long e = a; e < b; ++e) {
      const size_t base = (size_t)e * L;
      const int l = trimmed(M, elem_bytes, base, L);
      size_t s = 1;
      for (int t = 0; t < l; ++t) s += digits(elem(M, elem_bytes, base + t)) + (t ? 1 : 0);
      off[e + 1] = s;
    }
  });
  off[0] = head.size();
  for (long long e = 0; e < E; ++e) off[e + 1] += off[e];
  if (off[E] > cap) {
    set_last_error("text buffer of %zu bytes, %zu needed", cap, off[E]);
    return kInvalidArgument;
  }
  memcpy(out, head.data(), head.size());
  parallel_for(E, [&](long long a, long long b) {
    for (long long e = a; e < b; ++e) {
      const size_t base = (size_t)e * L;
      const int l = trimmed(M, elem_bytes, base, L);
      char* o = out + off[e];
      for (int t = 0; t < l; ++t) {
        if (t) *o++ = ' ';
        o = put_u64(o, elem(M, elem_bytes, base + t));
      }
      *o = '\n';
    }
  });
  if (written) *written = off[E];
  return kOk;
}

// header of a text matrix and the longest entry (trimmed, after reduction
// mod p): sizes the dense buffer for fpm_polmat_from_text
int fpm_polmat_text_dims(const char* text, size_t len, long long* p, int* m, int* n,
                         int* max_len) {
  if (!text && len) return kInvalidArgument;
  const std::vector<Line> lines = split_lines(text, len);
  long long P, M, N;
  FPM_TRY(header(text, lines, &P, &M, &N));
  if (p) *p = P;
  if (M < 0 || N < 0 || M > (1 << 30) || N > (1 << 30)) {
    set_last_error("matrix header m=%lld n=%lld", M, N);
    return kInvalidArgument;
  }
  if (m) *m = (int)M;
  if (n) *n = (int)N;
  if (P < 2) {
    set_last_error("modulus %lld out of range", P);
    return kOutOfRange;
  }
  const long long E = M * N;
  const long long have = std::min<long long>(E, (long long)lines.size() - 1);
  std::atomic<int> gmax{0}, bad{0};
  parallel_for(have, [&](long long a, long long b) {
    int mx = 0;
    bool ok = true;
    for (long long e = a; e < b && ok; ++e) {
      int cnt = 0, last = 0;
      ok = for_tokens(text, lines[1 + e], [&](const char* s, size_t l) {
        uint64_t v;
        if (!parse_mod(s, l, (uint64_t)P, &v)) return false;
        ++cnt;
        if (v) last = cnt;
        return true;
      });
      mx = std::max(mx, last);
    }
    int cur = gmax.load();
    while (mx > cur && !gmax.compare_exchange_weak(cur, mx)) {
    }
    if (!ok) bad.store(1);
  });
  if (bad.load()) {
    set_last_error("invalid literal in matrix body");
    return kInvalidArgument;
  }
  const int mx = gmax.load();
  if (max_len) *max_len = mx;
  return kOk;
}

// polmat_from_text into a dense host buffer (m*n*L, zero-padded; entries
// longer than L after trimming are an error)
int fpm_polmat_from_text(const char* text, size_t len, int elem_bytes, void* M, int L) {
  if ((elem_bytes != 4 && elem_bytes != 8) || L < 0) return kInvalidArgument;
  const std::vector<Line> lines = split_lines(text, len);
  long long P, Mr, Nc;
  FPM_TRY(header(text, lines, &P, &Mr, &Nc));
  if (P < 2 || (elem_bytes == 4 && P > (1LL << 32))) {
    set_last_error("modulus %lld does not fit %d-byte elements", P, elem_bytes);
    return kOutOfRange;
  }
  const long long E = Mr * Nc;
  if (E > 0 && L > 0) memset(M, 0, (size_t)E * L * elem_bytes);
  const long long have = std::min<long long>(E, (long long)lines.size() - 1);
  std::atomic<int> failed{0};
  parallel_for(have, [&](long long a, long long b) {
    for (long long e = a; e < b; ++e) {
      int t = 0, last = 0;
      const size_t base = (size_t)e * L;
      bool ok = for_tokens(text, lines[1 + e], [&](const char* s, size_t l) {
        uint64_t v;
        if (!parse_mod(s, l, (uint64_t)P, &v)) return false;
        if (v) {
          if (t >= L) return false;
          last = t + 1;
        }
        if (t < L) {
          if (elem_bytes == 4)
            ((uint32_t*)M)[base + t] = (uint32_t)v;
          else
            ((uint64_t*)M)[base + t] = v;
        }
        ++t;
        return true;
      });
      (void)last;
      if (!ok) failed.store(1);
    }
  });
  if (failed.load()) {
    set_last_error("invalid literal in matrix body, or an entry longer than %d", L);
    return kInvalidArgument;
  }
  return kOk;
}

}  // extern "C"
