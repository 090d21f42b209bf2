// small_path.cuh -- products of at most kSmallPairs term pairs in one CTA.
//
// Small products (expression powering's first steps, the reference's unit
// tests, service requests) are latency-bound: the multi-kernel paths spend
// 200-300 us in launches and host round trips on a few thousand pairs.  Here
// one CTA forms every pair's (compact key, row-major pair index) as one 64-bit
// sort word, bitonic-sorts them in shared memory, finds the runs of equal keys,
// lets one thread fold each run in increasing pair index (= increasing row i:
// the reference's order, merge.py:32-33, so doubles are bit-identical), drops
// zero sums (merge.py:63) and writes the compacted terms.  One launch, one
// host round trip.
#pragma once
#include "common.cuh"

namespace pgpu {

#ifndef PGPU_SMALL_PAIRS
#define PGPU_SMALL_PAIRS 16384
#endif
constexpr int kSmallPairs = PGPU_SMALL_PAIRS;  // 8 B sort word + 2 B head each, in shared memory
constexpr int kSmallThreads = 1024;
constexpr size_t kSmallSmem = kSmallPairs * 8 + (kSmallPairs + 8) * 2;

struct SmallArgs {
  const void* ak;  // compact keys (KT)
  const void* bk;
  const void* ac;
  const void* bc;
  uint32_t na, nb;
  uint64_t KL, KH;  // compact key range [KL, KH)
  int pbits;        // bits of the pair index in a sort word
  KeyPlan P;
  uint64_t* oexp;   // capacity na*nb
  uint64_t* ocoef;  // capacity na*nb*NL (f64: one word)
  unsigned long long* count;  // [0] terms written, [1] pairs formed
};

__device__ __forceinline__ uint32_t small_scan(uint32_t v, uint32_t* sh, uint32_t* total) {
  return block_excl_scan(v, sh, total);
}

// CK: 0 f64 (reference order), 1 int64, 2 int128; NL result limbs
template <typename KT, int NL, int CK>
__global__ void __launch_bounds__(kSmallThreads)
k_small_product(SmallArgs A) {
  extern __shared__ __align__(16) uint64_t small_smem[];
  uint64_t* sv = small_smem;                                            // [kSmallPairs]
  uint16_t* head = reinterpret_cast<uint16_t*>(small_smem + kSmallPairs);  // [kSmallPairs + 1]
  __shared__ uint32_t sh[33];
  __shared__ uint32_t nvalid_s, nseg_s;
  const KT* __restrict__ ak = reinterpret_cast<const KT*>(A.ak);
  const KT* __restrict__ bk = reinterpret_cast<const KT*>(A.bk);
  const uint32_t pairs = A.na * A.nb;
  uint32_t p2 = 1;
  while (p2 < pairs) p2 <<= 1;
  const uint64_t pmask = (1ull << A.pbits) - 1;
  // 1. sort words: (key << pbits) | pair index; pairs outside [KL, KH) sort last
  uint32_t nv = 0;
  for (uint32_t p = threadIdx.x; p < p2; p += blockDim.x) {
    uint64_t word = ~0ull;
    if (p < pairs) {
      const uint32_t i = p / A.nb, j = p - i * A.nb;
      const uint64_t key = (uint64_t)ak[i] + (uint64_t)bk[j];
      if (key >= A.KL && key < A.KH) {
        word = (key << A.pbits) | p;
        ++nv;
      }
    }
    sv[p] = word;
  }
  uint32_t nvalid;
  small_scan(nv, sh, &nvalid);
  __syncthreads();
  // 2. bitonic sort of sv[0, p2)
  for (uint32_t size = 2; size <= p2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t t = threadIdx.x; t < p2 / 2; t += blockDim.x) {
        const uint32_t lo = 2 * t - (t & (stride - 1));
        const uint32_t hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t x = sv[lo], y = sv[hi];
        if ((x > y) == up) {
          sv[lo] = y;
          sv[hi] = x;
        }
      }
      __syncthreads();
    }
  }
  // 3. run heads among the valid words, compacted into head[]
  {
    constexpr int C = kSmallPairs / kSmallThreads;
    const uint32_t c0 = threadIdx.x * C;
    uint32_t flags = 0, cnt = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const uint32_t q = c0 + c;
      const bool h = q < nvalid && (q == 0 || (sv[q] >> A.pbits) != (sv[q - 1] >> A.pbits));
      flags |= (h ? 1u : 0u) << c;
      cnt += h ? 1u : 0u;
    }
    uint32_t nseg;
    uint32_t pos = small_scan(cnt, sh, &nseg);
#pragma unroll
    for (int c = 0; c < C; ++c)
      if ((flags >> c) & 1u) head[pos++] = (uint16_t)(c0 + c);
    if (threadIdx.x == 0) {
      head[nseg] = (uint16_t)nvalid;  // nvalid <= kSmallPairs < 2^16
      nseg_s = nseg;
      nvalid_s = nvalid;
    }
  }
  __syncthreads();
  const uint32_t nseg = nseg_s;
  const uint32_t nvalid_all = nvalid_s;
  // 4. one thread per run, folded in increasing pair index (row order)
  uint32_t nzc = 0;
  uint64_t acc[kSmallPairs / kSmallThreads][NL];
  uint32_t nzm = 0;
#pragma unroll
  for (int u = 0; u < kSmallPairs / kSmallThreads; ++u) {
    const uint32_t s = threadIdx.x * (kSmallPairs / kSmallThreads) + u;
#pragma unroll
    for (int w = 0; w < NL; ++w) acc[u][w] = 0;
    if (s >= nseg) continue;
    const uint32_t q0 = head[s];
    const uint32_t q1 = s + 1 < nseg ? head[s + 1] : nvalid_all;
    bool nz;
    if constexpr (CK == 0) {
      double d = 0.0;
      for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t p = (uint32_t)(sv[q] & pmask);
        const uint32_t i = p / A.nb, j = p - i * A.nb;
        const double pr = __dmul_rn(reinterpret_cast<const double*>(A.ac)[i],
                                    reinterpret_cast<const double*>(A.bc)[j]);
        d = q == q0 ? pr : __dadd_rn(d, pr);
      }
      nz = d != 0.0;  // NaN kept, +-0 dropped (merge.py:63)
      acc[u][0] = (uint64_t)__double_as_longlong(d);
    } else {
      Limbs<NL> l;
      limbs_zero(l);
      for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t p = (uint32_t)(sv[q] & pmask);
        const uint32_t i = p / A.nb, j = p - i * A.nb;
        limbs_add(l, imul<NL, CK>(load_icoef<CK>(A.ac, (int64_t)i), load_icoef<CK>(A.bc, (int64_t)j)));
      }
      nz = limbs_nonzero(l);
#pragma unroll
      for (int w = 0; w < NL; ++w) acc[u][w] = l.w[w];
    }
    if (nz) {
      nzm |= 1u << u;
      ++nzc;
    }
  }
  // 5. compaction in run order
  uint32_t nnz;
  uint32_t pos = small_scan(nzc, sh, &nnz);
#pragma unroll
  for (int u = 0; u < kSmallPairs / kSmallThreads; ++u) {
    if (!((nzm >> u) & 1u)) continue;
    const uint32_t s = threadIdx.x * (kSmallPairs / kSmallThreads) + u;
    A.oexp[pos] = expand_key(sv[head[s]] >> A.pbits, A.P);
#pragma unroll
    for (int w = 0; w < NL; ++w) A.ocoef[(uint64_t)pos * NL + w] = acc[u][w];
    ++pos;
  }
  if (threadIdx.x == 0) {
    A.count[0] = nnz;
    A.count[1] = nvalid_all;  // pairs inside [KL, KH)
  }
}

}  // namespace pgpu
