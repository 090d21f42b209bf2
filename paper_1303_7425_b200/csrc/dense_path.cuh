// dense_path.cuh -- the fused fast path for products whose result exponents
// are dense in compact key space (Fateman-type benchmarks).
//
// The paper's two steps (Alg. 1, PAPER.md; reference parmul.py:64-109):
//
//   symbolic  D1 k_symbolic   every pair's compact key marks one byte of a
//                             sumset bytemap (idempotent byte stores: no
//                             atomics, order-free).  Replaces the exponent
//                             sort/merge of heap_merge/tree_merge
//                             (merge.py:42-62, 113-131): the result exponent
//                             set is exactly the marked keys, ascending.
//             D2 k_words      bytemap -> bit words + exclusive rank prefix
//                             (device scan) + the ascending output key list.
//   numeric   D3 k_edges_multi  per interval bound, each row's column bound
//                             (find_edge, split.py:131-166) by two-pointer walks.
//             D4 k_numeric    one CTA per (interval, row block).  Interval =
//                             D consecutive output terms.  Each warp owns a
//                             private accumulator copy in shared memory and
//                             walks one row at a time with lanes on consecutive
//                             columns: keys of one row are distinct, so no two
//                             lanes touch the same slot -- no atomics, no locks
//                             (the paper's independent-term property).  The
//                             slot of a pair is its output rank (bit words +
//                             prefix).  Warps' copies are folded by one owner
//                             thread per output term.
//             D5 k_fold       (row-blocked intervals) one owner per output
//                             term sums the row blocks' partials, tests zero
//                             (merge.py:63) and writes the exponent.
#pragma once
#include "common.cuh"
#include "scan.cuh"

namespace pgpu {

// ---- D1 ---------------------------------------------------------------------
constexpr int kSymRows = 64;     // rows per CTA tile
constexpr int kSymCols = 4096;   // columns per CTA tile (B keys staged in smem)

template <typename KT>
__global__ void __launch_bounds__(256)
k_symbolic(const KT* __restrict__ ak, const KT* __restrict__ bk, const uint32_t* __restrict__ rlo,
           const uint32_t* __restrict__ rhi, uint32_t na, uint32_t nb, uint64_t R0,
           uint8_t* __restrict__ bytemap) {
  __shared__ KT sb[kSymCols];
  const uint32_t c0 = blockIdx.x * kSymCols;
  const uint32_t c1 = min(c0 + kSymCols, nb);
  const uint32_t r0 = blockIdx.y * kSymRows;
  const uint32_t r1 = min(r0 + kSymRows, na);
  // rows' column ranges shrink leftwards with i: the tile is empty unless
  // [rlo[r1-1], rhi[r0]) meets [c0, c1)
  if (rhi[r0] <= c0 || rlo[r1 - 1] >= c1) return;
  for (uint32_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) sb[c - c0] = bk[c];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t i = r0 + w; i < r1; i += blockDim.x >> 5) {
    uint32_t lo = max(rlo[i], c0), hi = min(rhi[i], c1);
    uint64_t a = (uint64_t)ak[i] - R0;
    for (uint32_t j = lo + lane; j < hi; j += 32) bytemap[a + (uint64_t)sb[j - c0]] = 1;
  }
}

// ---- D2 ---------------------------------------------------------------------
// word w covers keys [32w, 32w+32) of the span
struct WordGen {
  const uint8_t* bytemap;
  uint64_t span;
  __device__ uint32_t mask(uint64_t w) const {
    uint64_t k0 = w * 32;
    uint32_t m = 0;
    if (k0 + 32 <= span) {
      const uint4* p = reinterpret_cast<const uint4*>(bytemap + k0);
      uint4 x = p[0], y = p[1];
      uint32_t v[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t t = v[q];
        // byte b of word q -> bit 4q+b
        uint32_t nib = (t & 0xffu ? 1u : 0u) | (t & 0xff00u ? 2u : 0u) |
                       (t & 0xff0000u ? 4u : 0u) | (t & 0xff000000u ? 8u : 0u);
        m |= nib << (4 * q);
      }
    } else {
      for (uint64_t k = k0; k < span; ++k)
        if (bytemap[k]) m |= 1u << (k - k0);
    }
    return m;
  }
  __device__ uint32_t operator()(uint64_t w) const { return __popc(mask(w)); }
};

template <typename OKT>
struct WordOut {
  WordGen gen;
  uint32_t* bits;
  uint32_t* prefix;
  OKT* okey;
  uint64_t R0;
  __device__ void operator()(uint64_t w, uint32_t ex, uint32_t v) const {
    uint32_t m = gen.mask(w);
    bits[w] = m;
    prefix[w] = ex;
    uint32_t r = ex;
    while (m) {
      int b = __ffs(m) - 1;
      m &= m - 1;
      okey[r++] = (OKT)(R0 + w * 32 + b);
    }
  }
};

// ---- D3 ---------------------------------------------------------------------
// E[t*na + i] = #{j : ak[i] + bk[j] < bound_t}, bound_t = okey[t*D] (t < T),
// bound_T = R1.  One thread walks kEdgeRun consecutive rows: a binary search
// for the first row, then the column pointer only moves left.
constexpr int kEdgeRun = 16;

template <typename KT>
__device__ __forceinline__ uint64_t interval_bound(const KT* okey, uint32_t t, uint32_t T, uint32_t D,
                                                   uint64_t R1) {
  return t < T ? (uint64_t)okey[(uint64_t)t * D] : R1;
}

template <typename KT>
__global__ void __launch_bounds__(256)
k_edges_multi(const KT* __restrict__ ak, uint32_t na, const KT* __restrict__ bk, uint32_t nb,
              const KT* __restrict__ okey, uint32_t T, uint32_t D, uint64_t R1,
              uint32_t* __restrict__ E, uint32_t t_off) {
  const uint32_t t = blockIdx.y + t_off;
  const uint64_t K = interval_bound(okey, t, T, D, R1);
  const uint32_t nchunks = (na + kEdgeRun - 1) / kEdgeRun;
  for (uint32_t ch = blockIdx.x * blockDim.x + threadIdx.x; ch < nchunks;
       ch += gridDim.x * blockDim.x) {
    uint32_t i0 = ch * kEdgeRun, i1 = min(i0 + kEdgeRun, na);
    uint32_t c = count_below(bk, nb, (uint64_t)ak[i0], K);
    uint32_t* e = E + (uint64_t)t * na;
    e[i0] = c;
    for (uint32_t i = i0 + 1; i < i1; ++i) {
      uint64_t ai = ak[i];
      while (c > 0 && ai + (uint64_t)bk[c - 1] >= K) --c;
      e[i] = c;
    }
  }
}

// ---- D4 ---------------------------------------------------------------------
constexpr int kNumThreads = 256;
constexpr int kNumWarps = kNumThreads / 32;

// Shared-memory accumulator words: acc[word][warp][slot] (u32), NW words per
// term (int), or a double per (warp, slot) for f64.
template <int NW, int CK>
__device__ __forceinline__ void words_of_product(const ICoef& a, const ICoef& b, uint32_t (&p)[NW]) {
  constexpr int NL = (NW + 1) / 2;
  Limbs<NL> r = imul<NL, CK>(a, b);
#pragma unroll
  for (int k = 0; k < NW; ++k) p[k] = (uint32_t)(r.w[k >> 1] >> (32 * (k & 1)));
}

template <int NW>
__device__ __forceinline__ void smem_add_words(uint32_t* acc, uint32_t stride, const uint32_t (&p)[NW]) {
  uint64_t c = 0;
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    uint64_t s = (uint64_t)acc[k * stride] + p[k] + c;
    acc[k * stride] = (uint32_t)s;
    c = s >> 32;
  }
}

template <typename KT>
__device__ __forceinline__ uint32_t rank_of(uint64_t klocal, const uint32_t* __restrict__ bits,
                                            const uint32_t* __restrict__ prefix) {
  uint64_t w = klocal >> 5;
  uint32_t m = __ldg(bits + w) & ((1u << (klocal & 31)) - 1u);
  return __ldg(prefix + w) + __popc(m);
}

// Accumulate one (interval, row block) unit.  Output: if `final_out`, the
// owner thread writes the finished term; else the unit's partial words.
template <typename KT, int NW, int CK>
__global__ void __launch_bounds__(kNumThreads)
k_numeric_int(const KT* __restrict__ ak, const KT* __restrict__ bk, const void* __restrict__ ac,
              const void* __restrict__ bc, uint32_t na, const uint32_t* __restrict__ E,
              const uint32_t* __restrict__ bits, const uint32_t* __restrict__ prefix, uint64_t R0,
              uint32_t nout, uint32_t D, uint32_t R, uint32_t* __restrict__ partial,
              const KT* __restrict__ okey, KeyPlan P, int nl, uint64_t* __restrict__ oexp,
              uint64_t* __restrict__ ocoef, uint32_t* __restrict__ onz) {
  extern __shared__ uint32_t sacc[];  // [NW][kNumWarps][D]
  const uint32_t t = blockIdx.x / R, r = blockIdx.x % R;
  const uint32_t base = t * D;
  const uint32_t dcount = min(D, nout - base);
  const uint32_t stride = kNumWarps * D;
  for (uint32_t k = threadIdx.x; k < NW * stride; k += blockDim.x) sacc[k] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t rb0 = (uint32_t)((uint64_t)na * r / R), rb1 = (uint32_t)((uint64_t)na * (r + 1) / R);
  const uint32_t* e0 = E + (uint64_t)t * na;
  const uint32_t* e1 = e0 + na;
  uint32_t* my = sacc + w * D;
  // warps take 32-row groups round robin; inside a group, one row at a time
  for (uint32_t g = rb0 + w * 32; g < rb1; g += kNumWarps * 32) {
    uint32_t i = g + lane;
    uint32_t lo = 0, hi = 0;
    if (i < rb1) {
      lo = e0[i];
      hi = e1[i];
    }
    unsigned todo = __ballot_sync(0xffffffffu, hi > lo);
    while (todo) {
      int src = __ffs(todo) - 1;
      todo &= todo - 1;
      uint32_t ri = g + src;
      uint32_t jlo = __shfl_sync(0xffffffffu, lo, src);
      uint32_t jhi = __shfl_sync(0xffffffffu, hi, src);
      uint64_t a = (uint64_t)ak[ri] - R0;
      ICoef ca = load_icoef<CK>(ac, ri);
      for (uint32_t j = jlo + lane; j < jhi; j += 32) {
        uint64_t kl = a + (uint64_t)bk[j];
        uint32_t slot = rank_of<KT>(kl, bits, prefix) - base;
        ICoef cb = load_icoef<CK>(bc, j);
        uint32_t p[NW];
        words_of_product<NW, CK>(ca, cb, p);
        smem_add_words<NW>(my + slot, stride, p);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  // one owner thread per output slot folds the warps' copies
  for (uint32_t s = threadIdx.x; s < dcount; s += blockDim.x) {
    uint32_t v[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) v[k] = 0;
#pragma unroll 1
    for (int q = 0; q < kNumWarps; ++q) {
      uint32_t p[NW];
#pragma unroll
      for (int k = 0; k < NW; ++k) p[k] = sacc[k * stride + q * D + s];
      uint64_t c = 0;
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        uint64_t x = (uint64_t)v[k] + p[k] + c;
        v[k] = (uint32_t)x;
        c = x >> 32;
      }
    }
    if (R == 1) {
      uint32_t o = base + s;
      uint64_t nzv = 0;
      for (int k = 0; k < nl; ++k) {
        uint32_t lo = 2 * k < NW ? v[2 * k] : (uint32_t)((int32_t)v[NW - 1] >> 31);
        uint32_t hi = 2 * k + 1 < NW ? v[2 * k + 1] : (uint32_t)((int32_t)v[NW - 1] >> 31);
        uint64_t limb = (uint64_t)lo | ((uint64_t)hi << 32);
        ocoef[(uint64_t)o * nl + k] = limb;
      }
#pragma unroll
      for (int k = 0; k < NW; ++k) nzv |= v[k];
      onz[o] = nzv ? 1u : 0u;
      oexp[o] = expand_key((uint64_t)okey[o], P);
    } else {
      uint32_t* dst = partial + ((uint64_t)blockIdx.x * D + s) * NW;
#pragma unroll
      for (int k = 0; k < NW; ++k) dst[k] = v[k];
    }
  }
}

template <typename KT>
__global__ void __launch_bounds__(kNumThreads)
k_numeric_f64(const KT* __restrict__ ak, const KT* __restrict__ bk, const double* __restrict__ ac,
              const double* __restrict__ bc, uint32_t na, const uint32_t* __restrict__ E,
              const uint32_t* __restrict__ bits, const uint32_t* __restrict__ prefix, uint64_t R0,
              uint32_t nout, uint32_t D, uint32_t R, double* __restrict__ partial,
              const KT* __restrict__ okey, KeyPlan P, uint64_t* __restrict__ oexp,
              double* __restrict__ ocoef, uint32_t* __restrict__ onz) {
  extern __shared__ double sdacc[];  // [kNumWarps][D]
  const uint32_t t = blockIdx.x / R, r = blockIdx.x % R;
  const uint32_t base = t * D;
  const uint32_t dcount = min(D, nout - base);
  for (uint32_t k = threadIdx.x; k < kNumWarps * D; k += blockDim.x) sdacc[k] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t rb0 = (uint32_t)((uint64_t)na * r / R), rb1 = (uint32_t)((uint64_t)na * (r + 1) / R);
  const uint32_t* e0 = E + (uint64_t)t * na;
  const uint32_t* e1 = e0 + na;
  double* my = sdacc + w * D;
  for (uint32_t g = rb0 + w * 32; g < rb1; g += kNumWarps * 32) {
    uint32_t i = g + lane;
    uint32_t lo = 0, hi = 0;
    if (i < rb1) {
      lo = e0[i];
      hi = e1[i];
    }
    unsigned todo = __ballot_sync(0xffffffffu, hi > lo);
    while (todo) {
      int src = __ffs(todo) - 1;
      todo &= todo - 1;
      uint32_t ri = g + src;
      uint32_t jlo = __shfl_sync(0xffffffffu, lo, src);
      uint32_t jhi = __shfl_sync(0xffffffffu, hi, src);
      uint64_t a = (uint64_t)ak[ri] - R0;
      double ca = __ldg(ac + ri);
      for (uint32_t j = jlo + lane; j < jhi; j += 32) {
        uint64_t kl = a + (uint64_t)bk[j];
        uint32_t slot = rank_of<KT>(kl, bits, prefix) - base;
        my[slot] = __dadd_rn(my[slot], __dmul_rn(ca, __ldg(bc + j)));
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < dcount; s += blockDim.x) {
    double v = 0.0;
#pragma unroll 1
    for (int q = 0; q < kNumWarps; ++q) v = __dadd_rn(v, sdacc[q * D + s]);
    if (R == 1) {
      uint32_t o = base + s;
      ocoef[o] = v;
      onz[o] = v != 0.0 ? 1u : 0u;
      oexp[o] = expand_key((uint64_t)okey[o], P);
    } else {
      partial[(uint64_t)blockIdx.x * D + s] = v;
    }
  }
}

// ---- D5 ---------------------------------------------------------------------
template <typename KT, int NW>
__global__ void __launch_bounds__(256)
k_fold_int(const uint32_t* __restrict__ partial, uint32_t nout, uint32_t D, uint32_t R,
           const KT* __restrict__ okey, KeyPlan P, int nl, uint64_t* __restrict__ oexp,
           uint64_t* __restrict__ ocoef, uint32_t* __restrict__ onz) {
  uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= nout) return;
  uint32_t t = o / D, s = o % D;
  uint32_t v[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) v[k] = 0;
  for (uint32_t r = 0; r < R; ++r) {
    const uint32_t* src = partial + ((uint64_t)(t * R + r) * D + s) * NW;
    uint64_t c = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      uint64_t x = (uint64_t)v[k] + src[k] + c;
      v[k] = (uint32_t)x;
      c = x >> 32;
    }
  }
  uint64_t nzv = 0;
  for (int k = 0; k < nl; ++k) {
    uint32_t lo = 2 * k < NW ? v[2 * k] : (uint32_t)((int32_t)v[NW - 1] >> 31);
    uint32_t hi = 2 * k + 1 < NW ? v[2 * k + 1] : (uint32_t)((int32_t)v[NW - 1] >> 31);
    ocoef[(uint64_t)o * nl + k] = (uint64_t)lo | ((uint64_t)hi << 32);
  }
#pragma unroll
  for (int k = 0; k < NW; ++k) nzv |= v[k];
  onz[o] = nzv ? 1u : 0u;
  oexp[o] = expand_key((uint64_t)okey[o], P);
}

template <typename KT>
__global__ void __launch_bounds__(256)
k_fold_f64(const double* __restrict__ partial, uint32_t nout, uint32_t D, uint32_t R,
           const KT* __restrict__ okey, KeyPlan P, uint64_t* __restrict__ oexp,
           double* __restrict__ ocoef, uint32_t* __restrict__ onz) {
  uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= nout) return;
  uint32_t t = o / D, s = o % D;
  double v = 0.0;
  for (uint32_t r = 0; r < R; ++r) v = __dadd_rn(v, partial[(uint64_t)(t * R + r) * D + s]);
  ocoef[o] = v;
  onz[o] = v != 0.0 ? 1u : 0u;
  oexp[o] = expand_key((uint64_t)okey[o], P);
}

}  // namespace pgpu
