// common.cuh -- shared device code: order-preserving exponent keys, exact
// integer limb arithmetic, row edges (FindEdge) and a device-wide scan.
//
// Reference anchors:
//   * packed exponent layout / raw u64 addition licensed by check_product_fits
//     (core.py:154-196, core.py:365-385);
//   * find_edge's per-row column bounds (split.py:131-166): here every row's
//     bound is lower_bound(B, K - a_i) in compact key space;
//   * coefficient accumulation `acc = a_i*b_j; acc += ...` (merge.py:49-58) with
//     Python's unbounded ints replaced by fixed-width two's-complement limbs
//     whose width the host proves sufficient (see pgpu_mul).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Checked build (-DPGPU_CHECKED, lib/libpolymul_b200_checked.so): device-side
// bounds assertions on every shared-memory slot, table and output index the
// kernels compute (a failed one traps and the call returns PGPU_ECUDA).  The
// product build compiles them out.
#ifdef PGPU_CHECKED
#include <cassert>
#define PGPU_ASSERT(c) assert(c)
#else
#define PGPU_ASSERT(c) ((void)0)
#endif

namespace pgpu {

constexpr int kMaxFields = 15;

// Compaction of a packed exponent word into a short key.  Each field keeps its
// exact value but is narrowed to bit_length(max_a_f + max_b_f) bits; field order
// (MSB first) is unchanged, so unsigned order of keys equals unsigned order of
// the packed sums for every realisable sum, and compact(a)+compact(b) ==
// compact(a+b) because no field sum can carry.  Under grlex the last variable
// is implied by the degree and is dropped from the key.
struct KeyPlan {
  int nf;
  int order;                 // 0 grlex, 1 lex
  int dropped;               // field recomputed from the degree, or -1
  int kbits;                 // significant key bits
  int shift[kMaxFields];
  int keep[kMaxFields];
  int cpos[kMaxFields];
  uint64_t mask[kMaxFields];  // packed-field mask (after shifting down)
  uint64_t cmask[kMaxFields]; // compact-field mask
};

__host__ __device__ __forceinline__ uint64_t compact_word(uint64_t e, const KeyPlan& P) {
  uint64_t k = 0;
#pragma unroll 1
  for (int f = 0; f < P.nf; ++f)
    if (P.keep[f]) k |= ((e >> P.shift[f]) & P.mask[f]) << P.cpos[f];
  return k;
}

// Inverse of compact_word on realisable sums (the output exponent of a key).
__device__ __forceinline__ uint64_t expand_key(uint64_t k, const KeyPlan& P) {
  uint64_t e = 0, deg = 0, vars = 0;
#pragma unroll 1
  for (int f = 0; f < P.nf; ++f) {
    if (!P.keep[f]) continue;
    uint64_t v = (k >> P.cpos[f]) & P.cmask[f];
    e |= v << P.shift[f];
    if (P.order == 0) {
      if (f == 0) deg = v; else vars += v;
    }
  }
  if (P.dropped >= 0) e |= (deg - vars) << P.shift[P.dropped];
  return e;
}

// ---------------------------------------------------------------------------
// Exact integer coefficients.  Operands: CK=1 int64, CK=2 int128 (lo,hi limbs).
// A product is formed modulo 2^(64*NL); sums are accumulated modulo 2^(64*NL).
// The host proves |every output coefficient| < 2^(64*NL-1), so the final
// two's-complement value is exact even though partial sums may wrap.
// ---------------------------------------------------------------------------
template <int NL>
struct Limbs {
  uint64_t w[NL];
};

template <int NL>
__device__ __forceinline__ void limbs_zero(Limbs<NL>& x) {
#pragma unroll
  for (int k = 0; k < NL; ++k) x.w[k] = 0;
}

template <int NL>
__device__ __forceinline__ void limbs_add(Limbs<NL>& acc, const Limbs<NL>& p) {
  if constexpr (NL == 1) {
    acc.w[0] += p.w[0];
  } else if constexpr (NL == 2) {
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;"
        : "+l"(acc.w[0]), "+l"(acc.w[1]) : "l"(p.w[0]), "l"(p.w[1]));
  } else {
    asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %5;"
        : "+l"(acc.w[0]), "+l"(acc.w[1]), "+l"(acc.w[2])
        : "l"(p.w[0]), "l"(p.w[1]), "l"(p.w[2]));
  }
}

template <int NL>
__device__ __forceinline__ bool limbs_nonzero(const Limbs<NL>& x) {
  uint64_t o = 0;
#pragma unroll
  for (int k = 0; k < NL; ++k) o |= x.w[k];
  return o != 0;
}

// Operand coefficient in sign-extended 3-limb form (only the needed limbs used).
struct ICoef {
  uint64_t x0, x1, x2;
};

template <int CK>
__device__ __forceinline__ ICoef load_icoef(const void* base, int64_t idx) {
  ICoef c;
  if constexpr (CK == 1) {
    int64_t v = __ldg(reinterpret_cast<const long long*>(base) + idx);
    c.x0 = (uint64_t)v;
    c.x1 = c.x2 = (uint64_t)(v >> 63);
  } else {
    const unsigned long long* p = reinterpret_cast<const unsigned long long*>(base) + 2 * idx;
    c.x0 = __ldg(p);
    c.x1 = __ldg(p + 1);
    c.x2 = (uint64_t)((int64_t)c.x1 >> 63);
  }
  return c;
}

// (a*b) mod 2^(64*NL) from sign-extended operands.
template <int NL, int CK>
__device__ __forceinline__ Limbs<NL> imul(const ICoef& a, const ICoef& b) {
  Limbs<NL> r;
  if constexpr (NL == 1) {
    r.w[0] = a.x0 * b.x0;
  } else if constexpr (CK == 1) {
    r.w[0] = a.x0 * b.x0;
    uint64_t hi = (uint64_t)__mul64hi((long long)a.x0, (long long)b.x0);
    r.w[1] = hi;
    if constexpr (NL == 3) r.w[2] = (uint64_t)((int64_t)hi >> 63);
  } else {
    // schoolbook, truncated: limb k collects a_i*b_j with i+j == k
    unsigned __int128 t00 = (unsigned __int128)a.x0 * b.x0;
    r.w[0] = (uint64_t)t00;
    unsigned __int128 t01 = (unsigned __int128)a.x0 * b.x1;
    unsigned __int128 t10 = (unsigned __int128)a.x1 * b.x0;
    unsigned __int128 s1 = (t00 >> 64) + (uint64_t)t01;
    s1 += (uint64_t)t10;
    r.w[1] = (uint64_t)s1;
    if constexpr (NL == 3) {
      uint64_t s2 = (uint64_t)(s1 >> 64) + (uint64_t)(t01 >> 64) + (uint64_t)(t10 >> 64) +
                    a.x0 * b.x2 + a.x1 * b.x1 + a.x2 * b.x0;
      r.w[2] = s2;
    }
  }
  return r;
}

// ---------------------------------------------------------------------------
// Row edges: number of columns j with ak[i] + bk[j] < K (B keys ascending).
// ---------------------------------------------------------------------------
template <typename KT>
__device__ __forceinline__ uint32_t count_below(const KT* __restrict__ bk, uint32_t nb,
                                                uint64_t ai, uint64_t K) {
  if (K <= ai) return 0;
  uint64_t t = K - ai;  // want #{j : bk[j] < t}
  uint32_t lo = 0, hi = nb;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if ((uint64_t)bk[mid] < t) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// Warp / block scan helpers.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Exclusive block scan for blockDim.x <= 1024 (multiple of 32).
// `sh` needs 33 elements.  Returns the exclusive prefix; *total = block sum.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* sh, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T s = lane < nw ? sh[lane] : T(0);
    T si = warp_incl_scan(s);
    if (lane < nw) sh[lane] = si - s;
    if (lane == nw - 1) sh[32] = si;
  }
  __syncthreads();
  T r = sh[wid] + inc - v;
  *total = sh[32];
  __syncthreads();
  return r;
}

}  // namespace pgpu
