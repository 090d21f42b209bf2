// dense_path.cuh -- the fused fast path for products whose result exponents
// are dense in compact key space (Fateman-type benchmarks).
//
// The paper's two steps (Alg. 1, PAPER.md; reference parmul.py:64-109):
//
//   symbolic  D0 k_head_scan  runs of consecutive keys in each operand
//             D1 k_symbolic   the sumset bitmap as a union of run-pair
//                             intervals (each key of the window set once,
//                             order-free).  Replaces the exponent sort/merge
//                             of heap_merge/tree_merge (merge.py:42-62,
//                             113-131): the result exponent set is exactly the
//                             set bits, ascending.
//             D2 device_scan  bit words -> exclusive rank prefix + the
//                             ascending output key list.
//   numeric   D4 k_numeric    one CTA per (row block, segment of consecutive
//                             intervals).  Interval = D consecutive output
//                             terms.  Each row keeps a cursor, so its run in
//                             the next interval is found by walking forward
//                             (find_edge, split.py:131-166, amortised to one
//                             comparison per pair).  Each warp owns a private
//                             accumulator copy in shared memory and walks one
//                             row at a time with lanes on consecutive columns:
//                             keys of one row are distinct, so no two lanes
//                             touch the same slot -- no atomics, no locks (the
//                             paper's independent-term property).  A pair's
//                             slot is its output rank (bit words + prefix, or a
//                             per-interval shared-memory table).  One owner
//                             thread per output term folds the warps' copies.
//             D5 k_fold       one owner per output term sums the row blocks'
//                             partials, tests zero (merge.py:63) and writes the
//                             exponent.
#pragma once
#include <type_traits>
#ifndef PGPU_UNROLL
#define PGPU_UNROLL 1
#endif
#ifndef PGPU_NUM_WARPS
#define PGPU_NUM_WARPS 16
#endif
#include "common.cuh"
#include "scan.cuh"

namespace pgpu {

// ---- D1 ---------------------------------------------------------------------
// Compact keys of dense operands come in runs of consecutive values (the last
// field counting up: each Fateman n=30 operand has 5,456 runs of ~8.5 terms),
// and the keys of (a-run p) x (b-run q) are exactly the interval
// [first_p + first_q, last_p + last_q].  The sumset is the union of those
// intervals: 29.8M for F30 instead of 2.15e9 pair keys (operands without runs
// degrade to one interval per pair).  One CTA per window of ww*32 keys of
// [R0, R1): the a-runs that can reach the window (binary search), for each
// the b-runs whose interval meets it (binary search), the clipped interval's
// bits set in shared memory (atomicOr on its partial end words, plain stores
// of all-ones words: idempotent, order-free), then the window's words written
// once to the global bitmap (one owner per word: no atomics, no memset).
template <typename KT>
__device__ __forceinline__ uint32_t lower_bound_key(const KT* __restrict__ s, uint32_t n, uint64_t v) {
  uint32_t lo = 0, hi = n;  // first i with s[i] >= v
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((uint64_t)__ldg(s + mid) < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void sym_mark(uint32_t* wb, uint32_t s, uint32_t e) {  // bits [s, e), s < e
  const uint32_t ws = s >> 5, we = (e - 1) >> 5;
  const uint32_t ms = ~0u << (s & 31), me = ~0u >> (31 - ((e - 1) & 31));
  if (ws == we) {
    atomicOr(wb + ws, ms & me);
    return;
  }
  atomicOr(wb + ws, ms);
  for (uint32_t w = ws + 1; w < we; ++w) wb[w] = ~0u;
  atomicOr(wb + we, me);
}

// Lanes take consecutive a-runs (similar keys: similar b-run ranges, little
// divergence).  (Measured on F30: contiguous a-run shares per thread with
// galloping bounds, or a block-scanned even split of the intervals, were
// 1.2-1.4x slower.)
constexpr int kSymThreads = 256;

template <typename KT>
__global__ void __launch_bounds__(kSymThreads)
k_symbolic(const KT* __restrict__ af, const KT* __restrict__ al, const uint32_t* __restrict__ nra_p,
           const KT* __restrict__ bf, const KT* __restrict__ bl, const uint32_t* __restrict__ nrb_p,
           uint64_t R0, uint64_t R1, uint32_t ww, uint32_t* __restrict__ bits) {
  extern __shared__ uint32_t wb[];  // ww words
  const uint64_t K0 = R0 + (uint64_t)blockIdx.x * ww * 32;
  if (K0 >= R1) return;
  const uint64_t K1 = K0 + (uint64_t)ww * 32 < R1 ? K0 + (uint64_t)ww * 32 : R1;
  for (uint32_t q = threadIdx.x; q < ww; q += blockDim.x) wb[q] = 0;
  const uint32_t nra = *nra_p, nrb = *nrb_p;
  const uint64_t bmin = bf[0], bmax = bl[nrb - 1];
  // a-runs that can reach the window: last + bmax >= K0 and first + bmin < K1
  const uint32_t p0 = lower_bound_key(al, nra, K0 > bmax ? K0 - bmax : 0);
  const uint32_t p1 = lower_bound_key(af, nra, K1 > bmin ? K1 - bmin : 0);
  __syncthreads();
  for (uint32_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    const uint64_t a0 = af[p], a1 = al[p];
    // b-runs meeting the window with this a-run: last_q >= K0 - a1, first_q < K1 - a0
    const uint32_t q0 = lower_bound_key(bl, nrb, K0 > a1 ? K0 - a1 : 0);
    const uint32_t q1 = lower_bound_key(bf, nrb, K1 > a0 ? K1 - a0 : 0);
    for (uint32_t q = q0; q < q1; ++q) {
      const uint64_t klo = max(a0 + (uint64_t)__ldg(bf + q), K0);
      const uint64_t khi = min(a1 + (uint64_t)__ldg(bl + q) + 1, K1);
      if (klo < khi) sym_mark(wb, (uint32_t)(klo - K0), (uint32_t)(khi - K0));
    }
  }
  __syncthreads();
  uint32_t* dst = bits + (K0 - R0) / 32;
  const uint32_t nw = (uint32_t)((K1 - K0 + 31) / 32);
  for (uint32_t q = threadIdx.x; q < nw; q += blockDim.x) dst[q] = wb[q];
}

// ---- D2 ---------------------------------------------------------------------
// word w covers keys [R0 + 32w, R0 + 32w + 32)
struct WordGen {
  const uint32_t* bits;
  __device__ uint32_t mask(uint64_t w) const { return bits[w]; }
  __device__ uint32_t operator()(uint64_t w) const { return __popc(bits[w]); }
};

template <typename OKT>
struct WordOut {
  WordGen gen;
  uint32_t* prefix;
  OKT* okey;
  uint64_t R0;
  uint64_t span_cap;  // key span (checked build: marks stay inside it)
  __device__ void operator()(uint64_t w, uint32_t ex, uint32_t v) const {
    uint32_t m = gen.mask(w);
    prefix[w] = ex;
    uint32_t r = ex;
    while (m) {
      int b = __ffs(m) - 1;
      m &= m - 1;
      PGPU_ASSERT(R0 + w * 32 + b < R0 + span_cap);
      okey[r++] = (OKT)(R0 + w * 32 + b);
    }
  }
};

// ---- D3/D4 -------------------------------------------------------------------
// Interval t = output ranks [t*D, (t+1)*D); bound_t = okey[t*D], bound_T = R1.
template <typename KT>
__device__ __forceinline__ uint64_t interval_bound(const KT* okey, uint32_t t, uint32_t T, uint32_t D,
                                                   uint64_t R1) {
  return t < T ? (uint64_t)okey[(uint64_t)t * D] : R1;
}

constexpr int kNumWarps = PGPU_NUM_WARPS;
constexpr int kNumThreads = kNumWarps * 32;
constexpr uint32_t kTbl = 8192;      // keys covered by the shared-memory slot table
constexpr int kCursorRun = 8;        // rows per thread in the cursor initialisation
#ifndef PGPU_ACC_KB
#define PGPU_ACC_KB 80
#endif
constexpr size_t kAccBytes = PGPU_ACC_KB * 1024;
constexpr int kUnroll = PGPU_UNROLL;       // independent columns per lane per step
#ifndef PGPU_ROW_SELECT
#define PGPU_ROW_SELECT 1
#endif
#ifndef PGPU_ROW_CLAIM
#define PGPU_ROW_CLAIM 32
#endif
constexpr int kRowClaim = PGPU_ROW_CLAIM;  // rows a warp claims at a time (<= 32; 32 measured best)

// Accumulator geometry.  NW = words of a finished term.  CB = 1: the term is
// held as 4 word planes plus a one-byte carry counter (nonnegative products
// below 2^128 and a proven bound <= 136 bits: at most 255 carries per copy),
// else as NW word planes.  D = terms per interval.
template <int NW, int CB>
struct Geo {
  static constexpr int NP = CB ? 4 : NW;                 // u32 planes (4 = two u64 planes)
  static constexpr uint32_t D =
      (uint32_t)(kAccBytes / (kNumWarps * (NP * 4 + CB))) / 32 * 32 - 32;
  static constexpr uint32_t DP = D + 32;                 // + one pad slot per lane
  static constexpr uint32_t stride = kNumWarps * DP;     // words between planes
  static constexpr size_t tbl_off = (size_t)NP * stride * 4 + (CB ? (stride + 15) / 16 * 16 : 0);
  static constexpr size_t smem = tbl_off + kTbl * 2;
};

// MODE: 0 f64 (NW = 2: one double), 1 int64 with all coefficients >= 0
//       (unsigned products, carry into words >= 4 only when it happens),
//       2 int64 signed, 3 int128 signed.
struct NumArgs {
  const void* ak;
  const void* bk;    // padded with kUnroll*32 entries past nb
  const void* ac;
  const void* bc;
  uint32_t na, nb;
  const uint32_t* bits;
  const uint32_t* prefix;
  uint64_t R0, R1;
  const void* okey;
  uint32_t nout, D, T, R, S;
  uint32_t* cursor;  // [S][na]: next column of each row for this interval segment
  void* nextkey;     // [S][na]: key at that column (KT; all-ones when exhausted)
  void* partial;     // [T][R][D][NW] words (R > 1)
  int nl;
  uint64_t* oexp;
  uint64_t* ocoef;
  uint32_t* onz;
  uint32_t* unit_ctr;  // persistent CTAs: next unit to claim (zeroed before launch)
  const uint32_t* act;  // [T][2]: rows [act_lo, act_hi) that can meet interval t (k_active_rows)
};

// Finished term: NW words -> nl sign-extended u64 limbs + nonzero flag.
template <int NW, int MODE>
__device__ __forceinline__ void write_term(const NumArgs& A, uint32_t o, const uint32_t (&v)[NW]) {
  const uint32_t ext = MODE == 1 ? 0u : (uint32_t)((int32_t)v[NW - 1] >> 31);
  uint32_t nzv = 0;
#pragma unroll
  for (int k = 0; k < NW; ++k) nzv |= v[k];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (k < A.nl) {
      const uint32_t lo = 2 * k < NW ? v[2 * k < NW ? 2 * k : 0] : ext;
      const uint32_t hi = 2 * k + 1 < NW ? v[2 * k + 1 < NW ? 2 * k + 1 : 0] : ext;
      A.ocoef[(uint64_t)o * A.nl + k] = (uint64_t)lo | ((uint64_t)hi << 32);
    }
  }
  A.onz[o] = nzv ? 1u : 0u;
}

// acc[k*stride] += p (little-endian words, modulo 2^(32 NW))
template <int NW, uint32_t STRIDE>
__device__ __forceinline__ void add_words(uint32_t* a, const uint32_t (&p)[NW]) {
  uint32_t v[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) v[k] = a[k * STRIDE];
  if constexpr (NW == 2) {
    asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(v[0]), "+r"(v[1]) : "r"(p[0]), "r"(p[1]));
  } else if constexpr (NW == 3) {
    asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
        : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]) : "r"(p[0]), "r"(p[1]), "r"(p[2]));
  } else if constexpr (NW == 4) {
    asm("add.cc.u32 %0, %0, %4;\n\taddc.cc.u32 %1, %1, %5;\n\taddc.cc.u32 %2, %2, %6;\n\t"
        "addc.u32 %3, %3, %7;"
        : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3])
        : "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3]));
  } else if constexpr (NW == 5) {
    asm("add.cc.u32 %0, %0, %5;\n\taddc.cc.u32 %1, %1, %6;\n\taddc.cc.u32 %2, %2, %7;\n\t"
        "addc.cc.u32 %3, %3, %8;\n\taddc.u32 %4, %4, %9;"
        : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4])
        : "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3]), "r"(p[4]));
  } else {
    asm("add.cc.u32 %0, %0, %6;\n\taddc.cc.u32 %1, %1, %7;\n\taddc.cc.u32 %2, %2, %8;\n\t"
        "addc.cc.u32 %3, %3, %9;\n\taddc.cc.u32 %4, %4, %10;\n\taddc.u32 %5, %5, %11;"
        : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5])
        : "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3]), "r"(p[4]), "r"(p[5]));
  }
#pragma unroll
  for (int k = 0; k < NW; ++k) a[k * STRIDE] = v[k];
}

// Unsigned 128-bit product into 4 word planes; the carry out of bit 128 bumps
// the slot's byte counter (rare: only when the copy crosses a 2^128 multiple).
template <uint32_t STRIDE>
__device__ __forceinline__ void add_unsigned128(uint32_t* a, uint8_t* carry, uint64_t lo, uint64_t hi) {
  uint32_t v0 = a[0], v1 = a[STRIDE], v2 = a[2 * STRIDE], v3 = a[3 * STRIDE], cy;
  asm("add.cc.u32 %0, %0, %5;\n\taddc.cc.u32 %1, %1, %6;\n\taddc.cc.u32 %2, %2, %7;\n\t"
      "addc.cc.u32 %3, %3, %8;\n\taddc.u32 %4, 0, 0;"
      : "+r"(v0), "+r"(v1), "+r"(v2), "+r"(v3), "=r"(cy)
      : "r"((uint32_t)lo), "r"((uint32_t)(lo >> 32)), "r"((uint32_t)hi), "r"((uint32_t)(hi >> 32)));
  a[0] = v0;
  a[STRIDE] = v1;
  a[2 * STRIDE] = v2;
  a[3 * STRIDE] = v3;
  if (cy) *carry += 1;
}

#ifndef PGPU_MAD_CHAIN
#define PGPU_MAD_CHAIN 1
#endif

#ifndef PGPU_FOLD_ZERO
#define PGPU_FOLD_ZERO 0
#endif
constexpr bool kFoldZero = PGPU_FOLD_ZERO;

// Ballot of a warp that is converged by construction (every call site runs
// with all 32 lanes): the raw vote avoids the divergence check and branch
// the intrinsic adds inside the hot loop.
__device__ __forceinline__ uint32_t warp_ballot(bool p) {
  uint32_t r;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tvote.sync.ballot.b32 %0, q, 0xffffffff;\n\t}"
               : "=r"(r) : "r"((uint32_t)p));
  return r;
}

// Profiling build (-DPGPU_NPROF=1): CTA cycles per phase of k_numeric (thread
// 0, barrier to barrier) and row-visit / step / pair counts.
#ifndef PGPU_NPROF
#define PGPU_NPROF 0
#endif
#if PGPU_NPROF
__device__ unsigned long long g_nprof[8];
#define NPROF_T(k)                                        \
  if (threadIdx.x == 0) {                                 \
    const long long now_ = clock64();                     \
    atomicAdd(&g_nprof[k], (unsigned long long)(now_ - tprev)); \
    tprev = now_;                                         \
  }
#else
#define NPROF_T(k)
#endif

template <typename KT>
__device__ __forceinline__ uint32_t rank_of(uint64_t klocal, const uint32_t* __restrict__ bits,
                                            const uint32_t* __restrict__ prefix) {
  uint64_t w = klocal >> 5;
  uint32_t m = __ldg(bits + w) & ((1u << (klocal & 31)) - 1u);
  return __ldg(prefix + w) + __popc(m);
}

// One CTA = (row block r, interval segment s).  Intervals of the segment are
// processed in ascending order; each row keeps a cursor (first column whose key
// is >= the current interval's lower bound), so a row's run in interval t is
// found by walking forward from its cursor -- no per-interval edge search.
template <typename KT, int NW, int MODE, int CB>
__device__ __forceinline__ void numeric_unit(const NumArgs& A, const uint32_t unit) {
  using G = Geo<NW, CB>;
  constexpr uint32_t D = G::D;
  constexpr uint32_t DP = G::DP;
  constexpr uint32_t STRIDE = G::stride;
  constexpr int NP = G::NP;
  extern __shared__ __align__(16) uint32_t smem_u32[];
  __shared__ uint32_t row_ctr;
  uint32_t* acc = smem_u32;                                        // [NP][W][D]
  uint8_t* cbyte = reinterpret_cast<uint8_t*>(acc + NP * STRIDE);  // [W][D] (CB)
  uint16_t* tbl = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(smem_u32) + G::tbl_off);
  const KT* __restrict__ ak = (const KT*)A.ak;
  const KT* __restrict__ bk = (const KT*)A.bk;
  const KT* __restrict__ okey = (const KT*)A.okey;
  const uint32_t r = unit % A.R, s = unit / A.R;
  const uint32_t t_begin = (uint32_t)((uint64_t)A.T * s / A.S);
  const uint32_t t_end = (uint32_t)((uint64_t)A.T * (s + 1) / A.S);
  const uint32_t rb0 = (uint32_t)((uint64_t)A.na * r / A.R);
  const uint32_t rb1 = (uint32_t)((uint64_t)A.na * (r + 1) / A.R);
  uint32_t* cur = A.cursor + (uint64_t)s * A.na;
  KT* nk = (KT*)A.nextkey + (uint64_t)s * A.na;
  const KT kInf = (KT)~(KT)0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t nb = A.nb;
  if (t_begin >= t_end) return;
#if PGPU_NPROF
  long long tprev = clock64();
  unsigned long long visits = 0, steps = 0, npairs = 0;
#endif
  {  // cursors at the segment's first bound: binary search for a run's first
     // row, then a galloping search back from the previous row's cursor (the
     // count is non-increasing in i; consecutive rows of a degree layer can
     // differ by thousands of columns, so a linear walk is not bounded)
    const uint64_t K0 = interval_bound(okey, t_begin, A.T, D, A.R1);
    const uint32_t nrow = rb1 - rb0;
    for (uint32_t ch = threadIdx.x; ch * kCursorRun < nrow; ch += blockDim.x) {
      uint32_t i0 = rb0 + ch * kCursorRun, i1 = min(i0 + kCursorRun, rb1);
      uint32_t c = count_below(bk, nb, (uint64_t)ak[i0], K0);
      for (uint32_t i = i0; i < i1; ++i) {
        uint64_t ai = ak[i];
        if (i > i0 && c > 0 && ai + (uint64_t)bk[c - 1] >= K0) {
          // the count lies in [0, c - 1]: gallop down, then bisect the bracket
          uint32_t hi = c - 1, step = 1;
          while (hi >= step && ai + (uint64_t)bk[hi - step] >= K0) {
            hi -= step;
            step <<= 1;
          }
          uint32_t lo = hi >= step ? hi - step + 1 : 0;  // P(lo - 1) holds (or lo = 0)
          while (lo < hi) {  // first j in [lo, hi] with ai + bk[j] >= K0 (hi qualifies)
            const uint32_t mid = (lo + hi) >> 1;
            if (ai + (uint64_t)bk[mid] < K0) lo = mid + 1; else hi = mid;
          }
          c = lo;
        }
        PGPU_ASSERT(c == count_below(bk, nb, ai, K0));
        cur[i] = c;
        nk[i] = c < nb ? (KT)(ai + (uint64_t)bk[c]) : kInf;
      }
    }
  }
  __syncthreads();
  NPROF_T(0)
  for (uint32_t t = t_begin; t < t_end; ++t) {
    const uint64_t Klo = interval_bound(okey, t, A.T, D, A.R1);
    const uint64_t Khi = interval_bound(okey, t + 1, A.T, D, A.R1);
    const KT kmax = (KT)(Khi - 1);  // keys of the interval: [Klo, kmax]
    const uint32_t base = t * D;
    // rows that can meet the interval: a_i + b_0 < Khi (started) and
    // a_i + b_last >= Klo (not finished); a is ascending, so a contiguous span
    const uint32_t act_lo = max(rb0, __ldg(A.act + 2 * t)), act_hi = min(rb1, __ldg(A.act + 2 * t + 1));
    const uint32_t g_first = act_lo > rb0 ? (act_lo - rb0) & ~31u : 0u;  // 32-row groups from rb0
    const uint32_t dcount = min(D, A.nout - base);
    const bool use_tbl = (Khi - Klo) <= kTbl;
    if (threadIdx.x == 0) row_ctr = g_first;
    // the fold zeroes the copies it reads, so only a unit's first interval clears
    if (!kFoldZero || t == t_begin)
      for (uint32_t k = threadIdx.x; k < G::tbl_off / 4; k += blockDim.x) acc[k] = 0;
    if (use_tbl) {
      const uint64_t w0 = (Klo - A.R0) >> 5, w1 = (Khi - 1 - A.R0) >> 5;
      for (uint64_t wd = w0 + threadIdx.x; wd <= w1; wd += blockDim.x) {
        uint32_t m = __ldg(A.bits + wd);
        uint32_t rk = __ldg(A.prefix + wd) - base;
        while (m) {
          int b = __ffs(m) - 1;
          m &= m - 1;
          uint64_t k = A.R0 + wd * 32 + b;
          if (k >= Klo && k < Khi) {
            PGPU_ASSERT(k - Klo < kTbl && rk < D);
            tbl[k - Klo] = (uint16_t)rk;
          }
          ++rk;
        }
      }
    }
    __syncthreads();
    uint32_t* my = acc + w * DP;
    // one step: kUnroll columns per lane of row (akr, a0/ad) from cursor c; invalid
    // lanes add into their private pad slot so the step has no divergent branch
    const uint64_t span_t = Khi - 1 - Klo;
    auto step = [&](const KT akr, const uint64_t a0, const double ad, const uint32_t ri,
                    const uint32_t c, auto tbl_mode) -> uint32_t {
      constexpr bool TBL = decltype(tbl_mode)::value;
      const uint32_t cl = c + lane;                // 32-bit column index: 2-instruction addresses
      const KT* __restrict__ bkr = bk + cl;        // row-relative: immediate offsets per u
      uint32_t nv = 0;
      uint32_t slot[kUnroll];
      bool okk[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint32_t j = c + lane + 32 * u;
        const KT key = (KT)(akr + bkr[32 * u]);  // bk is padded: the load is in bounds
        bool ok;
        uint32_t off;
        if constexpr (sizeof(KT) == 4) {
          // 32-bit keys: the interval bounds fit 32 bits too; an offset that
          // wraps (key below Klo) exceeds the span, so one compare suffices
          off = (uint32_t)key - (uint32_t)Klo;
          ok = j < nb && off <= (uint32_t)span_t;
        } else {
          const uint64_t dk = (uint64_t)key - Klo;  // wraps for keys below Klo
          ok = j < nb && dk <= span_t;
          off = (uint32_t)dk;
        }
        nv += __popc(warp_ballot(ok));
        uint32_t sl;
        if constexpr (TBL) {
          sl = tbl[min(off, kTbl - 1)];
        } else {
          sl = ok ? rank_of<KT>((uint64_t)key - A.R0, A.bits, A.prefix) - base : 0u;
        }
        slot[u] = ok ? sl : D + lane;
        PGPU_ASSERT(slot[u] < DP && (!ok || sl < D));
        okk[u] = ok;
      }
      if constexpr (MODE == 1 && CB) {
        const long long* __restrict__ bcr = reinterpret_cast<const long long*>(A.bc) + cl;
        const uint32_t al = (uint32_t)a0, ah = (uint32_t)(a0 >> 32);
        uint64_t* p64 = reinterpret_cast<uint64_t*>(acc) + 2 * w * DP;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint64_t b0 = okk[u] ? (uint64_t)__ldg(bcr + 32 * u) : 0ull;
          const uint32_t bl = (uint32_t)b0, bh = (uint32_t)(b0 >> 32);
          // one 16-byte element (4 words) per (warp, term): a single LDS.128/STS.128
          uint4* e = reinterpret_cast<uint4*>(p64) + slot[u];
          uint4 v = *e;
#if PGPU_MAD_CHAIN
          // acc += a*b as three multiply-add carry chains over the 32-bit words
          // (al*bl, ah*bh; al*bh << 32; ah*bl << 32); cy counts the wrap of
          // the 128-bit element (at most one: the product is below 2^128)
          uint32_t cy;
          asm("mad.lo.cc.u32  %0, %5, %7, %0;\n\t"
              "madc.hi.cc.u32 %1, %5, %7, %1;\n\t"
              "madc.lo.cc.u32 %2, %6, %8, %2;\n\t"
              "madc.hi.cc.u32 %3, %6, %8, %3;\n\t"
              "addc.u32       %4, 0, 0;\n\t"
              "mad.lo.cc.u32  %1, %5, %8, %1;\n\t"
              "madc.hi.cc.u32 %2, %5, %8, %2;\n\t"
              "addc.cc.u32    %3, %3, 0;\n\t"
              "addc.u32       %4, %4, 0;\n\t"
              "mad.lo.cc.u32  %1, %6, %7, %1;\n\t"
              "madc.hi.cc.u32 %2, %6, %7, %2;\n\t"
              "addc.cc.u32    %3, %3, 0;\n\t"
              "addc.u32       %4, %4, 0;"
              : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w), "=r"(cy)
              : "r"(al), "r"(ah), "r"(bl), "r"(bh));
#else
          // 64x64 -> 128 from four 32x32 -> 64 partial products
          const uint64_t t0 = (uint64_t)al * bl;
          const uint64_t t1 = (uint64_t)al * bh + (t0 >> 32);
          const uint64_t t2 = (uint64_t)ah * bl + (uint32_t)t1;
          const uint64_t t3 = (uint64_t)ah * bh + (t1 >> 32) + (t2 >> 32);
          const uint64_t lo = (t2 << 32) | (uint32_t)t0;
          uint64_t vx = ((uint64_t)v.y << 32) | v.x, vy = ((uint64_t)v.w << 32) | v.z;
          uint32_t cy;
          asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u32 %2, 0, 0;"
              : "+l"(vx), "+l"(vy), "=r"(cy) : "l"(lo), "l"(t3));
          v = make_uint4((uint32_t)vx, (uint32_t)(vx >> 32), (uint32_t)vy, (uint32_t)(vy >> 32));
#endif
          *e = v;
          if (cy) cbyte[w * DP + slot[u]] += 1;
        }
        return nv;
      } else {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint32_t j = okk[u] ? c + lane + 32 * u : 0u;
          if constexpr (MODE == 0) {
            double* d = reinterpret_cast<double*>(acc) + w * DP + slot[u];
            const double bv = okk[u] ? __ldg(reinterpret_cast<const double*>(A.bc) + j) : 0.0;
            *d = __dadd_rn(*d, __dmul_rn(ad, bv));
          } else if constexpr (MODE == 1) {
            const uint64_t b0 = okk[u] ? (uint64_t)__ldg(reinterpret_cast<const long long*>(A.bc) + j) : 0ull;
            const uint64_t lo = a0 * b0;
            uint32_t p[NW];
            const uint64_t hi = __umul64hi(a0, b0);
            const uint32_t w4[4] = {(uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32)};
#pragma unroll
            for (int k = 0; k < NW; ++k) p[k] = k < 4 ? w4[k] : 0u;
            add_words<NW, STRIDE>(my + slot[u], p);
          } else if constexpr (MODE == 2) {
            const uint64_t b0 = okk[u] ? (uint64_t)__ldg(reinterpret_cast<const long long*>(A.bc) + j) : 0ull;
            const uint64_t lo = a0 * b0;
            const uint64_t hi = (uint64_t)__mul64hi((long long)a0, (long long)b0);
            const uint32_t ext = (uint32_t)((int64_t)hi >> 63);
            const uint32_t w4[4] = {(uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32)};
            uint32_t p[NW];
#pragma unroll
            for (int k = 0; k < NW; ++k) p[k] = k < 4 ? w4[k] : ext;
            add_words<NW, STRIDE>(my + slot[u], p);
          } else {
            ICoef ca = load_icoef<2>(A.ac, ri);
            ICoef cb = load_icoef<2>(A.bc, j);
            if (!okk[u]) cb.x0 = cb.x1 = cb.x2 = 0;
            Limbs<3> pr = imul<3, 2>(ca, cb);
            uint32_t p[NW];
#pragma unroll
            for (int k = 0; k < NW; ++k) p[k] = (uint32_t)(pr.w[k >> 1] >> (32 * (k & 1)));
            add_words<NW, STRIDE>(my + slot[u], p);
          }
        }
        return nv;
      }
    };
    auto rows = [&](auto tbl_mode) {
      // integers: warps claim 32-row groups dynamically (one shared counter per
      // interval; exact sums do not depend on which copy a row lands in).
      // f64: static groups w, w + W, w + 2W, ... so every run folds the same
      // rows into the same warp copy and the sums are bit-identical run to run
      for (uint32_t it = 0;; ++it) {
        uint32_t g;
        if constexpr (MODE == 0) {
          g = rb0 + g_first + (w + it * kNumWarps) * kRowClaim;
        } else {
          g = 0;
          if (lane == 0) g = atomicAdd(&row_ctr, (uint32_t)kRowClaim);
          g = rb0 + __shfl_sync(0xffffffffu, g, 0);
        }
        if (g >= act_hi) break;
        const uint32_t i = g + lane;
        const bool rowok = lane < kRowClaim && i < rb1;
        uint32_t ci = rowok ? cur[i] : 0u;
        KT nki = rowok ? nk[i] : kInf;
        unsigned todo = __ballot_sync(0xffffffffu, (uint64_t)nki < Khi);
        if (!todo) continue;
        const KT akl = rowok ? ak[i] : (KT)0;
        uint64_t a0l = 0;
        double adl = 0.0;
        if constexpr (MODE == 0) adl = rowok ? __ldg(reinterpret_cast<const double*>(A.ac) + i) : 0.0;
        else if constexpr (MODE != 3) a0l = rowok ? (uint64_t)__ldg(reinterpret_cast<const long long*>(A.ac) + i) : 0ull;
        while (todo) {
          const int src = __ffs(todo) - 1;
          todo &= todo - 1;
          uint32_t c = __shfl_sync(0xffffffffu, ci, src);
          const KT akr = __shfl_sync(0xffffffffu, akl, src);
          const uint64_t a0 = __shfl_sync(0xffffffffu, a0l, src);
          const double ad = __shfl_sync(0xffffffffu, adl, src);
          for (;;) {
            const uint32_t nv = step(akr, a0, ad, g + src, c, tbl_mode);
            c += nv;
#if PGPU_NPROF
            ++steps;
            npairs += nv;
#endif
            if (nv < 32u * kUnroll) break;
          }
#if PGPU_NPROF
          ++visits;
#endif
#if PGPU_ROW_SELECT
          // branch-free: every lane computes, the row's owner keeps it
          const KT nxt = c < nb ? (KT)(akr + __ldg(bk + (c < nb ? c : 0))) : kInf;
          ci = lane == src ? c : ci;
          nki = lane == src ? nxt : nki;
#else
          if (lane == src) {
            ci = c;
            nki = c < nb ? (KT)(akr + bk[c]) : kInf;
          }
          __syncwarp();
#endif
        }
        if (rowok) {
          cur[i] = ci;
          nk[i] = nki;
        }
      }
    };
    NPROF_T(1)
    if (use_tbl) rows(std::integral_constant<bool, true>{});
    else rows(std::integral_constant<bool, false>{});
    __syncthreads();
    NPROF_T(2)
    // one owner thread per output slot folds the warps' private copies
    for (uint32_t sl = threadIdx.x; sl < dcount; sl += blockDim.x) {
      const uint32_t o = base + sl;
      if constexpr (MODE == 0) {
        const double* dacc = reinterpret_cast<const double*>(acc);
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < kNumWarps; ++q) v = __dadd_rn(v, dacc[q * DP + sl]);
        if constexpr (kFoldZero) {
#pragma unroll
          for (int q = 0; q < kNumWarps; ++q) reinterpret_cast<double*>(acc)[q * DP + sl] = 0.0;
        }
        if (A.R == 1) {
          reinterpret_cast<double*>(A.ocoef)[o] = v;
          A.onz[o] = v != 0.0 ? 1u : 0u;
        } else {
          reinterpret_cast<double*>(A.partial)[((uint64_t)t * A.R + r) * D + sl] = v;
        }
      } else {
        auto word_of = [&](int k, uint32_t e) -> uint32_t {
          if constexpr (CB) {
            const uint64_t* p64 = reinterpret_cast<const uint64_t*>(acc);  // [W][DP]{lo,hi}
            if (k < 2) return (uint32_t)(p64[2 * e] >> (32 * k));
            if (k < 4) return (uint32_t)(p64[2 * e + 1] >> (32 * (k - 2)));
            return k == 4 ? (uint32_t)cbyte[e] : 0u;
          } else {
            return k < NP ? acc[k * STRIDE + e] : 0u;
          }
        };
        uint32_t v[NW];
#pragma unroll
        for (int k = 0; k < NW; ++k) v[k] = word_of(k, sl);
#pragma unroll
        for (int q = 1; q < kNumWarps; ++q) {
          uint32_t pw[NW];
#pragma unroll
          for (int k = 0; k < NW; ++k) pw[k] = word_of(k, q * DP + sl);
          uint64_t cy = 0;
#pragma unroll
          for (int k = 0; k < NW; ++k) {
            uint64_t x = (uint64_t)v[k] + pw[k] + cy;
            v[k] = (uint32_t)x;
            cy = x >> 32;
          }
        }
        if constexpr (kFoldZero) {
#pragma unroll
          for (int q = 0; q < kNumWarps; ++q) {
            const uint32_t e = q * DP + sl;
            if constexpr (CB) {
              reinterpret_cast<ulonglong2*>(acc)[e] = make_ulonglong2(0ull, 0ull);
              cbyte[e] = 0;
            } else {
#pragma unroll
              for (int k = 0; k < NP; ++k) acc[k * STRIDE + e] = 0u;
            }
          }
        }
        if (A.R == 1) {
          write_term<NW, MODE>(A, o, v);
        } else {
          uint32_t* dst = reinterpret_cast<uint32_t*>(A.partial) + (((uint64_t)t * A.R + r) * D + sl) * NW;
#pragma unroll
          for (int k = 0; k < NW; ++k) dst[k] = v[k];
        }
      }
    }
    // with kFoldZero the next interval's table build needs no barrier here: the
    // barrier after it orders this fold before the next interval's rows
    if (!kFoldZero) __syncthreads();
    NPROF_T(3)
  }
#if PGPU_NPROF
  if (lane == 0) {
    atomicAdd(&g_nprof[4], visits);
    atomicAdd(&g_nprof[5], steps);
    atomicAdd(&g_nprof[6], npairs);
  }
#endif
}

// Persistent CTAs (one per resident slot) claim (row block, segment) units in
// key order from a counter: no partial last wave, and the light units at the
// top of the key range finish the grid.
#ifndef PGPU_PERSISTENT
#define PGPU_PERSISTENT 1
#endif
// Two CTAs per SM are resident either way (their accumulators fill shared
// memory), so the register budget is 64 per thread, not the 40 ptxas picks
// for a bare 512-thread bound (which spilled the f64 and 3-4 plane modes).
#ifndef PGPU_NUMERIC_MINB
#define PGPU_NUMERIC_MINB 2
#endif
template <typename KT, int NW, int MODE, int CB>
__global__ void __launch_bounds__(kNumThreads, PGPU_NUMERIC_MINB)
k_numeric(NumArgs A) {
#if PGPU_PERSISTENT
  __shared__ uint32_t unit_s;
  for (;;) {
    if (threadIdx.x == 0) unit_s = atomicAdd(A.unit_ctr, 1u);
    __syncthreads();
    const uint32_t unit = unit_s;
    __syncthreads();
    if (unit >= A.R * A.S) return;
    numeric_unit<KT, NW, MODE, CB>(A, unit);
  }
#else
  numeric_unit<KT, NW, MODE, CB>(A, blockIdx.x);
#endif
}

// Active row span of every interval t: rows [lo, hi) whose run can meet
// [bound_t, bound_t+1) -- finished rows (a_i + b_last < Klo) and rows not
// yet started (a_i + b_0 >= Khi) are skipped by the numeric pass.
template <typename KT>
__global__ void __launch_bounds__(256)
k_active_rows(const KT* __restrict__ ak, uint32_t na, const KT* __restrict__ bk, uint32_t nb,
              const KT* __restrict__ okey, uint32_t T, uint32_t D, uint64_t R1, uint32_t* __restrict__ act) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const uint64_t Klo = interval_bound(okey, t, T, D, R1), Khi = interval_bound(okey, t + 1, T, D, R1);
  act[2 * t] = count_below(ak, na, (uint64_t)bk[nb - 1], Klo);
  act[2 * t + 1] = count_below(ak, na, (uint64_t)bk[0], Khi);
}

// ---- D5 ---------------------------------------------------------------------
// One owner per output term: sums the row blocks' partials, zero test
// (merge.py:63), output exponent from its key.
template <typename KT, int NW, int MODE>
__global__ void __launch_bounds__(256)
k_fold(NumArgs A, KeyPlan P) {
  const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= A.nout) return;
  const uint32_t t = o / A.D, sl = o % A.D;
  if (A.R > 1) {
    if constexpr (MODE == 0) {
      double v = 0.0;
      for (uint32_t r = 0; r < A.R; ++r)
        v = __dadd_rn(v, reinterpret_cast<const double*>(A.partial)[((uint64_t)t * A.R + r) * A.D + sl]);
      reinterpret_cast<double*>(A.ocoef)[o] = v;
      A.onz[o] = v != 0.0 ? 1u : 0u;
    } else {
      uint32_t v[NW];
#pragma unroll
      for (int k = 0; k < NW; ++k) v[k] = 0;
      for (uint32_t r = 0; r < A.R; ++r) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(A.partial) +
                              (((uint64_t)t * A.R + r) * A.D + sl) * NW;
        uint64_t cy = 0;
#pragma unroll
        for (int k = 0; k < NW; ++k) {
          uint64_t x = (uint64_t)v[k] + src[k] + cy;
          v[k] = (uint32_t)x;
          cy = x >> 32;
        }
      }
      write_term<NW, MODE>(A, o, v);
    }
  }
  A.oexp[o] = expand_key((uint64_t)((const KT*)A.okey)[o], P);
}

}  // namespace pgpu
