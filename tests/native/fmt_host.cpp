// Host build of csrc/text.cuh for the CPU test-suite (tests/test_text.py):
// the same formatting code the GPU runs, compiled with g++, checked against
// Python's own str(int) / repr(float).
#include "../../paper_1303_7425_b200/csrc/text.cuh"

using namespace pgpu::text;

extern "C" {

// repr() of n doubles, '\n'-terminated, into out; returns bytes written
int64_t fmt_doubles(const double* v, int64_t n, char* out) {
  int64_t at = 0;
  for (int64_t i = 0; i < n; ++i) {
    BufW w{out + at};
    put_double(w, v[i]);
    CountW c;
    put_double(c, v[i]);
    if (c.n != w.n) return -1 - i;  // counting and writing must agree
    at += w.n;
    out[at++] = '\n';
  }
  return at;
}

// str() of n nl-limb integers
int64_t fmt_ints(const uint64_t* limbs, int nl, int64_t n, char* out) {
  int64_t at = 0;
  for (int64_t i = 0; i < n; ++i) {
    BufW w{out + at};
    put_int(w, limbs + i * nl, nl);
    CountW c;
    put_int(c, limbs + i * nl, nl);
    if (c.n != w.n) return -1 - i;
    at += w.n;
    out[at++] = '\n';
  }
  return at;
}

// full PolyFile lines
int64_t fmt_lines(const uint64_t* exps, const void* coef, int64_t n, const LineSpec* s, char* out) {
  int64_t at = 0;
  for (int64_t i = 0; i < n; ++i) {
    BufW w{out + at};
    put_line(w, *s, exps[i], coef, (uint64_t)i);
    at += w.n;
  }
  return at;
}
}
