// prep.cuh -- operand statistics, key compaction, range thresholds, row edges
// and pair counting.
//
//   k_stats        per-field maxima (check_product_fits, core.py:365-385) and
//                  coefficient magnitudes (accumulator-width proof)
//   k_compact      packed word -> order-preserving short key (KeyPlan)
//   k_threshold    packed bound S -> smallest compact key of a realisable sum
//                  >= S (so split=/cluster ranges translate exactly)
//   k_edges        per-row column range of a key interval (find_edge,
//                  split.py:131-166, computed by binary search per row)
//   k_count_multi  cum[k] = #pairs below bounds[k] (count_ops, split.py:169-175)
#pragma once
#include "common.cuh"

namespace pgpu {

struct OperandStats {
  unsigned long long fmax[2][kMaxFields];
  unsigned int cbits[2];
  unsigned int unsorted[2];
  unsigned int negative[2];
  unsigned long long maxmag[2];  // bits of an upper bound (double) of max |c|
};

__device__ __forceinline__ int bitlen_u64(uint64_t x) { return x ? 64 - __clzll((long long)x) : 0; }

template <int CK>
__global__ void __launch_bounds__(256)
k_stats(const uint64_t* __restrict__ exps, const void* __restrict__ coef, int64_t n, KeyPlan P,
        OperandStats* st, int side, double* __restrict__ bsum) {
  const int nf = P.nf;
  __shared__ unsigned long long smax[kMaxFields];
  __shared__ double ssum[32];
  __shared__ unsigned int sbits, sunsorted, sneg;
  __shared__ unsigned long long smag;  // max magnitude (nonnegative doubles order as their bits)
  if (threadIdx.x < kMaxFields) smax[threadIdx.x] = 0;
  if (threadIdx.x == 0) { sbits = 0; sunsorted = 0; sneg = 0; smag = 0; }
  __syncthreads();
  unsigned long long lmax[kMaxFields];
#pragma unroll
  for (int f = 0; f < kMaxFields; ++f) lmax[f] = 0;
  unsigned int lbits = 0, lbad = 0, lneg = 0;
  double lsum = 0.0;  // upper bound of sum |c| (rounded up)
  double lmag = 0.0;  // upper bound of max |c|
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t e = exps[i];
    if (i > 0 && exps[i - 1] >= e) lbad = 1;
    if (e == ~0ull) lbad = 1;
#pragma unroll
    for (int f = 0; f < kMaxFields; ++f)
      if (f < nf) {
        unsigned long long v = (e >> P.shift[f]) & P.mask[f];
        lmax[f] = v > lmax[f] ? v : lmax[f];
      }
    if constexpr (CK == 1) {
      int64_t c = reinterpret_cast<const int64_t*>(coef)[i];
      if (c < 0) lneg = 1;
      uint64_t mag = c < 0 ? (uint64_t)(-(c + 1)) + 1 : (uint64_t)c;
      int b = bitlen_u64(mag);
      lbits = b > (int)lbits ? b : lbits;
      lsum = __dadd_ru(lsum, __ull2double_ru(mag));
      lmag = fmax(lmag, __ull2double_ru(mag));
    } else if constexpr (CK == 2) {
      const uint64_t* p = reinterpret_cast<const uint64_t*>(coef) + 2 * i;
      uint64_t lo = p[0], hi = p[1];
      if ((int64_t)hi < 0) lneg = 1;
      if ((int64_t)hi < 0) {  // magnitude of a negative 128-bit value
        lo = ~lo; hi = ~hi;
        lo += 1;
        if (lo == 0) hi += 1;
      }
      int b = hi ? 64 + bitlen_u64(hi) : bitlen_u64(lo);
      lbits = b > (int)lbits ? b : lbits;
      double m = __dadd_ru(__dmul_ru(__ull2double_ru(hi), 18446744073709551616.0),
                           __ull2double_ru(lo));
      lsum = __dadd_ru(lsum, m);
      lmag = fmax(lmag, m);
    }
  }
#pragma unroll
  for (int f = 0; f < kMaxFields; ++f) {
    if (f < nf) {  // warp max first: one shared atomic per warp and field
      unsigned long long v = lmax[f];
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, d);
        v = o > v ? o : v;
      }
      if ((threadIdx.x & 31) == 0 && v) atomicMax(&smax[f], v);
    }
  }
  if (lbits) atomicMax(&sbits, lbits);
  if (lbad) sunsorted = 1;
  if (lneg) sneg = 1;
  // block sum of the per-thread upper bounds (rounded up) and block max of the
  // magnitudes: one global atomic per block (one per thread serialised on a
  // single word and cost ~0.1 ms per operand)
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    lsum = __dadd_ru(lsum, __shfl_xor_sync(0xffffffffu, lsum, d));
    lmag = fmax(lmag, __shfl_xor_sync(0xffffffffu, lmag, d));
  }
  if ((threadIdx.x & 31) == 0) {
    ssum[threadIdx.x >> 5] = lsum;
    if (lmag > 0.0) atomicMax(&smag, (unsigned long long)__double_as_longlong(lmag));
  }
  __syncthreads();
  if (threadIdx.x == 0 && smag) atomicMax(&st->maxmag[side], smag);
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t = __dadd_ru(t, ssum[q]);
    bsum[blockIdx.x] = t;
  }
  if (threadIdx.x < nf && smax[threadIdx.x]) atomicMax(&st->fmax[side][threadIdx.x], smax[threadIdx.x]);
  if (threadIdx.x == 0) {
    if (sbits) atomicMax(&st->cbits[side], sbits);
    if (sunsorted) st->unsorted[side] = 1;
    if (sneg) st->negative[side] = 1;
  }
}

template <typename KT>
__global__ void __launch_bounds__(256)
k_compact(const uint64_t* __restrict__ exps, int64_t n, KeyPlan P, KT* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (KT)compact_word(exps[i], P);
}

// Smallest packed sum a_i + b_j >= S (ULLONG_MAX if none).  Compaction is
// order-preserving and additive on realisable sums, so its compact key is the
// smallest compact key of a pair at or above S; the host compacts it, which
// lets the thresholds ride the operand-statistics round trip.
__global__ void __launch_bounds__(256)
k_threshold(const uint64_t* __restrict__ aexp, uint32_t na, const uint64_t* __restrict__ bexp, uint32_t nb,
            uint64_t S, unsigned long long* out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long best = ~0ull;
  if (i < na) {
    uint32_t j = count_below<uint64_t>(bexp, nb, aexp[i], S);
    if (j < nb) best = (unsigned long long)aexp[i] + (unsigned long long)bexp[j];
  }
  for (int d = 16; d > 0; d >>= 1) {
    unsigned long long o = __shfl_xor_sync(0xffffffffu, best, d);
    best = o < best ? o : best;
  }
  __shared__ unsigned long long sbest;
  if (threadIdx.x == 0) sbest = ~0ull;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(&sbest, best);
  __syncthreads();
  if (threadIdx.x == 0 && sbest != ~0ull) atomicMin(out, sbest);
}

// The smallest and largest packed exponent of each operand.
__global__ void k_exp_ends(const uint64_t* __restrict__ aexp, uint32_t na, const uint64_t* __restrict__ bexp,
                           uint32_t nb, unsigned long long* ends) {
  if (threadIdx.x == 0) {
    ends[0] = aexp[0];
    ends[1] = aexp[na - 1];
    ends[2] = bexp[0];
    ends[3] = bexp[nb - 1];
  }
}

template <typename KT>
__global__ void __launch_bounds__(256)
k_edges(const KT* __restrict__ ak, uint32_t na, const KT* __restrict__ bk, uint32_t nb,
        uint64_t KL, uint64_t KH, uint32_t* __restrict__ rlo, uint32_t* __restrict__ rhi) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= na) return;
  uint64_t ai = ak[i];
  rlo[i] = count_below(bk, nb, ai, KL);
  rhi[i] = count_below(bk, nb, ai, KH);
}

// cum[k] += #{(i,j): ak[i]+bk[j] < bounds[k]}; grid.y indexes bounds.
template <typename KT>
__global__ void __launch_bounds__(256)
k_count_multi(const KT* __restrict__ ak, uint32_t na, const KT* __restrict__ bk, uint32_t nb,
              const uint64_t* __restrict__ bounds, unsigned long long* cum) {
  uint64_t K = bounds[blockIdx.y];
  unsigned long long c = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += gridDim.x * blockDim.x)
    c += count_below(bk, nb, (uint64_t)ak[i], K);
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cum + blockIdx.y, c);
}

// ends[0..3] = ak[0], ak[na-1], bk[0], bk[nb-1] (operands ascending)
struct LenGen {
  const uint32_t* lo;
  const uint32_t* hi;
  __device__ uint64_t operator()(uint64_t i) const { return (uint64_t)(hi[i] - lo[i]); }
};

struct OffOut {
  uint64_t* off;
  __device__ void operator()(uint64_t i, uint64_t ex, uint64_t) const { off[i] = ex; }
};

}  // namespace pgpu
