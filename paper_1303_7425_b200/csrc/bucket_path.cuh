// bucket_path.cuh -- sparse products: pairs written once, grouped per CTA.
//
// The sort path moves every pair record through the global radix sort (one
// histogram pass plus 4-5 read+write passes).  For sparse products such as
// Monagan-Pearce most of that traffic is avoidable: an output term only needs
// its own pairs, and a paper interval of a few hundred pairs fits in one
// CTA's shared memory.  So the key range is cut into *buckets* of fewer than
// kBucketCap pairs (paper intervals sized for a CTA, split.py:1-9: equal keys
// never straddle a bound) and
//
//   B1 k_bin_count ×2 fine bins: coarse bins of 2^s1 keys, each split into 2^r
//                     equal sub-bins of ~kBinTarget pairs (BinMap); counted
//                     with one atomic per run of equal bins in a warp (keys
//                     ascend along a row, so a warp's bins form runs)
//   B2 device_scan    bin offsets; buckets = runs of bins whose offsets share a
//                     window of kBucketHalf records, a larger bin on its own
//   B3 k_bin_scatter  the same walk writes (key - KL, i<<32|j) once, at
//                     offset(bin) + atomic run position: records of one bucket
//                     are contiguous
//   B4 k_bucket_reduce one CTA per bucket: coalesced record loads and
//                     coefficient products; keys hashed into a shared-memory
//                     table whose slots accumulate the exact sums (32-bit
//                     atomics with explicit carries; f64 atomics in fast
//                     mode); distinct keys ranked (counting rank, or bitonic
//                     above 256); nonzero terms (merge.py:63) appended to a
//                     staging run.  A bucket that is one large bin is reduced
//                     in dense mode over the bin's key window.
//   B5 k_bucket_gather bucket runs -> final positions (bucket order = key
//                     order), one warp per bucket
//
// DRAM traffic per pair: one record write + one record read (12-16 B each),
// against 5-6 read+write passes on the sort path.  The float-ordered mode
// (reference summation order) stays on the sort path.
#pragma once
#include "common.cuh"
#include "scan.cuh"

namespace pgpu {

#ifndef PGPU_BUCKET_CAP
#define PGPU_BUCKET_CAP 512
#endif
constexpr int kBucketCap = PGPU_BUCKET_CAP;  // pairs per bucket (max)
constexpr int kBucketHalf = kBucketCap / 2;
constexpr int kBucketTable = 2 * kBucketCap; // hash slots (load factor <= 1/2)
#ifndef PGPU_BUCKET_THREADS
#define PGPU_BUCKET_THREADS 256
#endif
constexpr int kBucketThreads = PGPU_BUCKET_THREADS;

// ---- B1 / B3: walk of a batch's pairs ----------------------------------------
// One warp per row, lanes on consecutive columns (as k_gen).  For each group of
// 32 columns: bin per lane, run heads where the bin changes, run lengths from
// the head mask.
struct BinRun {
  uint32_t bin;
  bool head;
  uint32_t len;      // run length (heads only)
  int head_lane;     // lane of this lane's run head
};

__device__ __forceinline__ BinRun bin_runs(uint32_t bin, bool valid, int lane) {
  BinRun r;
  r.bin = bin;
  const uint32_t prev = __shfl_up_sync(0xffffffffu, bin, 1);
  r.head = valid && (lane == 0 || prev != bin);
  const uint32_t H = __ballot_sync(0xffffffffu, r.head);
  const uint32_t V = __ballot_sync(0xffffffffu, valid);  // valid lanes are 0..popc-1
  const uint32_t above = lane == 31 ? 0u : (H & (0xffffffffu << (lane + 1)));
  const int end = above ? __ffs(above) - 1 : __popc(V);
  r.len = (uint32_t)(end - lane);
  const uint32_t below = H & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
  r.head_lane = below ? 31 - __clz(below) : 0;
  return r;
}

// Key -> fine bin.  Level 1: coarse bins of 2^s1 keys.  Level 2: coarse bin c
// is split into 2^r_c equal sub-bins so that each holds ~kBinTarget pairs
// (tab[c] = first fine bin << 5 | r_c); fine bins ascend with the key.
struct BinMap {
  int s1;
  const uint32_t* tab;  // null: level 1
  __device__ __forceinline__ uint32_t operator()(uint64_t key) const {
    const uint32_t c = (uint32_t)(key >> s1);
    if (!tab) return c;
    const uint32_t t = __ldg(tab + c);
    const int r = (int)(t & 31u);
    return (t >> 5) + (uint32_t)((key & ((1ull << s1) - 1ull)) >> (s1 - r));
  }
};

template <typename KT>
__global__ void __launch_bounds__(256)
k_bin_count(const KT* __restrict__ ak, const KT* __restrict__ bk, const uint32_t* __restrict__ rlo,
            const uint32_t* __restrict__ rhi, uint32_t na, uint64_t KL, BinMap map,
            uint32_t* __restrict__ hist) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < na; i += nwarps) {
    const uint32_t j0 = rlo[i], j1 = rhi[i];
    if (j0 >= j1) continue;
    const uint64_t ai = (uint64_t)ak[i] - KL;
    for (uint32_t jb = j0; jb < j1; jb += 32) {
      const uint32_t j = jb + lane;
      const bool valid = j < j1;
      const uint32_t bin = valid ? map(ai + (uint64_t)__ldg(bk + j)) : 0xffffffffu;
      const BinRun r = bin_runs(bin, valid, lane);
      if (r.head) atomicAdd(hist + bin, r.len);
    }
  }
}

template <typename KT>
__global__ void __launch_bounds__(256)
k_bin_scatter(const KT* __restrict__ ak, const KT* __restrict__ bk, const uint32_t* __restrict__ rlo,
              const uint32_t* __restrict__ rhi, uint32_t na, uint64_t KL, BinMap map,
              uint32_t* __restrict__ fill, KT* __restrict__ rkey, uint64_t* __restrict__ rid) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < na; i += nwarps) {
    const uint32_t j0 = rlo[i], j1 = rhi[i];
    if (j0 >= j1) continue;
    const uint64_t ai = (uint64_t)ak[i] - KL;
    for (uint32_t jb = j0; jb < j1; jb += 32) {
      const uint32_t j = jb + lane;
      const bool valid = j < j1;
      const uint64_t key = valid ? ai + (uint64_t)__ldg(bk + j) : 0;
      const uint32_t bin = valid ? map(key) : 0xffffffffu;
      const BinRun r = bin_runs(bin, valid, lane);
      uint32_t pos = 0;
      if (r.head) pos = atomicAdd(fill + bin, r.len);
      pos = __shfl_sync(0xffffffffu, pos, r.head_lane) + (uint32_t)(lane - r.head_lane);
      if (valid) {
        rkey[pos] = (KT)key;
        rid[pos] = ((uint64_t)i << 32) | j;
      }
    }
  }
}

// level-2 split of each coarse bin: 2^r sub-bins, r the least with count >> r <= target
constexpr uint32_t kBinTarget = kBucketCap / 8;
struct RefineGen {
  const uint32_t* hist1;
  int s1;
  __device__ __forceinline__ int r_of(uint64_t c) const {
    const uint32_t n = hist1[c];
    int r = 0;
    while ((n >> r) > kBinTarget && r < s1) ++r;
    return r;
  }
  __device__ uint32_t operator()(uint64_t c) const { return 1u << r_of(c); }
};
struct RefineOut {
  RefineGen g;
  uint32_t* tab;
  __device__ void operator()(uint64_t c, uint32_t ex, uint32_t) const {
    tab[c] = (ex << 5) | (uint32_t)g.r_of(c);
  }
};

// Buckets: maximal runs of bins whose offsets share a window of kBucketHalf
// records (< kBucketCap records each), cut around any bin larger than
// kBucketHalf, which becomes a bucket of its own (reduced in dense mode).
struct BStartGen {
  const uint32_t* size;    // records per bin
  const uint32_t* binoff;
  __device__ uint32_t operator()(uint64_t b) const {
    if (b == 0) return 1u;
    const bool big = size[b] > (uint32_t)kBucketHalf, big_prev = size[b - 1] > (uint32_t)kBucketHalf;
    return (big || big_prev || binoff[b] / kBucketHalf != binoff[b - 1] / kBucketHalf) ? 1u : 0u;
  }
};
struct BStartOut {
  uint32_t* bstart;
  __device__ void operator()(uint64_t b, uint32_t ex, uint32_t v) const {
    if (v) bstart[ex] = (uint32_t)b;
  }
};

// ---- B4 ---------------------------------------------------------------------
struct BucketArgs {
  const void* rkey;            // KT keys relative to KL
  const uint64_t* rid;         // i<<32 | j
  const uint32_t* binoff;      // nbins offsets
  const uint32_t* bstart;      // nbuckets+1 first bins
  uint32_t nbins, pairs;
  int s1;                      // bin map (dense-mode key window)
  const uint32_t* tab;
  const void* ac;
  const void* bc;
  uint64_t KL;
  KeyPlan P;
  uint64_t* sexp;              // staging terms (capacity scap)
  uint64_t* scoef;
  uint64_t scap;
  unsigned long long* sctr;    // staging bump counter
  uint64_t* bbase;             // per bucket: staging base
  uint32_t* bnnz;              // per bucket: nonzero terms
  uint32_t* overflow;
};

template <typename KT, int NL>
struct BucketSmem {
  uint32_t acc[kBucketTable][2 * NL]; // per hash slot (dense mode: per key): the sum
  KT hkey[kBucketTable];              // open-addressing key table
  uint64_t sortv[kBucketCap];         // key << 12 | slot, sorted by key
  uint32_t scan[kBucketTable];        // occupied-slot flags, then nonzero-term flags
  uint32_t sh[33];
  uint32_t ndist;
  unsigned long long base;
};

__device__ __forceinline__ uint32_t cas_key(uint32_t* p, uint32_t cmp, uint32_t v) {
  return atomicCAS(reinterpret_cast<unsigned int*>(p), cmp, v);
}
__device__ __forceinline__ uint64_t cas_key(uint64_t* p, uint64_t cmp, uint64_t v) {
  return atomicCAS(reinterpret_cast<unsigned long long*>(p), (unsigned long long)cmp,
                   (unsigned long long)v);
}

__device__ __forceinline__ uint32_t bucket_hash(uint64_t k) {
  return (uint32_t)((k * 0x9E3779B97F4A7C15ull) >> 40) & (kBucketTable - 1);
}

// Exact accumulation of an NL-limb two's-complement product into 2*NL 32-bit
// words with native shared-memory atomics: the carry out of each word is
// recovered from the returned old value and added into the next word, so the
// words hold the exact sum modulo 2^(64 NL) whatever the interleaving.
template <int NL>
__device__ __forceinline__ void acc_add(uint32_t* a, const Limbs<NL>& p) {
  uint32_t carry = 0;
#pragma unroll
  for (int w = 0; w < 2 * NL; ++w) {
    const uint32_t pw = (uint32_t)(p.w[w >> 1] >> (32 * (w & 1)));
    const uint32_t x = pw + carry;
    const uint32_t c1 = x < pw ? 1u : 0u;
    if (x == 0u) {
      carry = c1;
      continue;
    }
    const uint32_t old = atomicAdd(a + w, x);
    carry = c1 + ((uint32_t)(old + x) < old ? 1u : 0u);
  }
}

// exclusive scan of x[0, n) in place, C items per thread (n <= C * blockDim),
// visible to the whole block on return; returns the total
template <int C>
__device__ __forceinline__ uint32_t chunk_scan(uint32_t* x, uint32_t n, uint32_t* sh) {
  const uint32_t c0 = threadIdx.x * C;
  uint32_t loc[C], s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    loc[c] = c0 + c < n ? x[c0 + c] : 0u;
    s += loc[c];
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan(s, sh, &tot);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    if (c0 + c < n) x[c0 + c] = ex;
    ex += loc[c];
  }
  __syncthreads();  // other threads read x[] next
  return tot;
}

template <int NL, int CK>
__device__ __forceinline__ void add_product(const BucketArgs& A, uint32_t* acc, uint64_t id) {
  const uint64_t i = id >> 32, j = id & 0xffffffffu;
  if constexpr (CK == 0) {
    const double pr = __dmul_rn(__ldg(reinterpret_cast<const double*>(A.ac) + i),
                                __ldg(reinterpret_cast<const double*>(A.bc) + j));
    atomicAdd(reinterpret_cast<double*>(acc), pr);
  } else {
    acc_add<NL>(acc, imul<NL, CK>(load_icoef<CK>(A.ac, (int64_t)i), load_icoef<CK>(A.bc, (int64_t)j)));
  }
}

template <int NL, int CK>
__device__ __forceinline__ bool acc_nonzero(const uint32_t* acc) {
  if constexpr (CK == 0) {
    return __longlong_as_double((long long)(((uint64_t)acc[1] << 32) | acc[0])) != 0.0;  // NaN kept
  } else {
    uint32_t o = 0;
#pragma unroll
    for (int w = 0; w < 2 * NL; ++w) o |= acc[w];
    return o != 0;
  }
}

// Staging: one bump-allocated run per bucket; returns the run base, or ~0 on overflow
__device__ __forceinline__ unsigned long long bucket_alloc(const BucketArgs& A, uint32_t k,
                                                           uint32_t nnz, unsigned long long* sbase) {
  if (threadIdx.x == 0) {
    unsigned long long b = atomicAdd(A.sctr, (unsigned long long)nnz);
    if (b + nnz > A.scap) {
      *A.overflow = 1u;
      b = ~0ull;
    }
    *sbase = b;
    A.bbase[k] = b;
    A.bnnz[k] = nnz;
  }
  __syncthreads();
  return *sbase;
}

template <int NL>
__device__ __forceinline__ void write_term(const BucketArgs& A, uint64_t pos, uint64_t key,
                                           const uint32_t* acc) {
  A.sexp[pos] = expand_key(A.KL + key, A.P);
#pragma unroll
  for (int w = 0; w < NL; ++w)
    A.scoef[pos * NL + w] = ((uint64_t)acc[2 * w + 1] << 32) | acc[2 * w];
}

// Dense mode for a bucket that is one fine bin above the record bound (many
// pairs on few keys): accumulators indexed by key - window base.  The window
// is the bin's key range (2^(s1 - r) keys); one wider than the table sets the
// overflow flag and the batch takes the sort path.
template <typename KT, int NL, int CK>
__device__ void bucket_dense(const BucketArgs& A, BucketSmem<KT, NL>& S, uint32_t k,
                             const KT* __restrict__ rkey, const uint64_t* __restrict__ rid,
                             uint32_t n) {
  const uint64_t key0 = (uint64_t)rkey[0];
  const uint32_t t = A.tab[key0 >> A.s1];
  const int sh = A.s1 - (int)(t & 31u);
  const uint64_t wbase = (key0 >> sh) << sh;
  if (sh > 20 || (1u << sh) > (uint32_t)kBucketTable) {
    if (threadIdx.x == 0) {
      *A.overflow = 1u;
      A.bnnz[k] = 0;
    }
    return;
  }
  const uint32_t span = 1u << sh;
  for (uint32_t x = threadIdx.x; x < span * 2 * NL; x += blockDim.x) (&S.acc[0][0])[x] = 0;
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < n; q += blockDim.x)
    add_product<NL, CK>(A, S.acc[(uint64_t)rkey[q] - wbase], rid[q]);
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < span; x += blockDim.x) S.scan[x] = acc_nonzero<NL, CK>(S.acc[x]);
  __syncthreads();
  const uint32_t nnz = chunk_scan<kBucketTable / kBucketThreads>(S.scan, span, S.sh);
  const unsigned long long base = bucket_alloc(A, k, nnz, &S.base);
  if (base == ~0ull) return;
  for (uint32_t x = threadIdx.x; x < span; x += blockDim.x) {
    const uint32_t nxt = x + 1 < span ? S.scan[x + 1] : nnz;
    if (nxt != S.scan[x]) write_term<NL>(A, base + S.scan[x], wbase + x, S.acc[x]);
  }
}

// CK: 0 f64 (fast mode, NL = 1), 1 int64, 2 int128 operands; NL result limbs
template <typename KT, int NL, int CK>
__global__ void __launch_bounds__(kBucketThreads)
k_bucket_reduce(BucketArgs A) {
  constexpr int IPT = kBucketCap / kBucketThreads;
  constexpr int TPT = kBucketTable / kBucketThreads;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  BucketSmem<KT, NL>& S = *reinterpret_cast<BucketSmem<KT, NL>*>(smem_raw);
  const uint32_t k = blockIdx.x;
  const uint32_t b0 = A.bstart[k], b1 = A.bstart[k + 1];
  const uint32_t r0 = A.binoff[b0];
  const uint32_t r1 = b1 < A.nbins ? A.binoff[b1] : A.pairs;
  const uint32_t n = r1 - r0;
  const KT* __restrict__ rkey = reinterpret_cast<const KT*>(A.rkey) + r0;
  const uint64_t* __restrict__ rid = A.rid + r0;
  if (n > (uint32_t)kBucketCap) {  // one large fine bin: dense mode over its key window
    bucket_dense<KT, NL, CK>(A, S, k, rkey, rid, n);
    return;
  }
  const KT kEmpty = (KT)~(KT)0;
  // 1. records (coalesced) while the table is cleared
  KT key[IPT];
  uint64_t id[IPT];
#pragma unroll
  for (int u = 0; u < IPT; ++u) {
    const uint32_t q = threadIdx.x + u * kBucketThreads;
    key[u] = q < n ? rkey[q] : kEmpty;
    id[u] = q < n ? rid[q] : 0ull;
  }
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const uint32_t t = threadIdx.x + u * kBucketThreads;
    S.hkey[t] = kEmpty;
#pragma unroll
    for (int w = 0; w < 2 * NL; ++w) S.acc[t][w] = 0;
  }
  __syncthreads();
  // 2. slot per key (equal keys share a slot); the product goes straight into it
#pragma unroll
  for (int u = 0; u < IPT; ++u) {
    if (key[u] == kEmpty) continue;
    uint32_t h = bucket_hash((uint64_t)key[u]);
    for (;;) {
      const KT prev = cas_key(&S.hkey[h], kEmpty, key[u]);
      if (prev == kEmpty || prev == key[u]) break;
      h = (h + 1) & (kBucketTable - 1);
    }
    add_product<NL, CK>(A, S.acc[h], id[u]);
  }
  __syncthreads();
  // 3. occupied slots, compacted in slot order
  {
    const uint32_t t0 = threadIdx.x * TPT;
#pragma unroll
    for (int u = 0; u < TPT; ++u) S.scan[t0 + u] = S.hkey[t0 + u] != kEmpty ? 1u : 0u;
  }
  const uint32_t nd = chunk_scan<TPT>(S.scan, kBucketTable, S.sh);
  {
    const uint32_t t0 = threadIdx.x * TPT;
#pragma unroll
    for (int u = 0; u < TPT; ++u) {
      const uint32_t t = t0 + u;
      const KT kk = S.hkey[t];
      if (kk != kEmpty) S.sortv[S.scan[t]] = ((uint64_t)kk << 12) | t;
    }
  }
  __syncthreads();
  // 4. distinct keys in key order
  if (nd <= kBucketThreads) {
    // few distinct keys (the common case): rank = number of smaller keys
    uint64_t mine = 0;
    uint32_t rank = 0;
    if (threadIdx.x < nd) {
      mine = S.sortv[threadIdx.x];
      for (uint32_t x = 0; x < nd; ++x) rank += S.sortv[x] < mine ? 1u : 0u;
    }
    __syncthreads();
    if (threadIdx.x < nd) S.sortv[rank] = mine;
    __syncthreads();
  } else {
    uint32_t p2 = 1;
    while (p2 < nd) p2 <<= 1;
    for (uint32_t t = nd + threadIdx.x; t < p2; t += blockDim.x) S.sortv[t] = ~0ull;
    __syncthreads();
    for (uint32_t size = 2; size <= p2; size <<= 1) {
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t t = threadIdx.x; t < p2 / 2; t += blockDim.x) {
          const uint32_t lo = 2 * t - (t & (stride - 1));
          const uint32_t hi = lo + stride;
          const bool up = (lo & size) == 0;
          const uint64_t x = S.sortv[lo], y = S.sortv[hi];
          if ((x > y) == up) {
            S.sortv[lo] = y;
            S.sortv[hi] = x;
          }
        }
        __syncthreads();
      }
    }
  }
  // 5. nonzero sums (merge.py:63) in key order -> staging
  for (uint32_t r = threadIdx.x; r < nd; r += blockDim.x)
    S.scan[r] = acc_nonzero<NL, CK>(S.acc[S.sortv[r] & 0xfff]) ? 1u : 0u;
  __syncthreads();
  const uint32_t nnz = chunk_scan<IPT>(S.scan, nd, S.sh);
  const unsigned long long base = bucket_alloc(A, k, nnz, &S.base);
  if (base == ~0ull) return;
  for (uint32_t r = threadIdx.x; r < nd; r += blockDim.x) {
    const uint32_t nxt = r + 1 < nd ? S.scan[r + 1] : nnz;
    if (nxt != S.scan[r]) write_term<NL>(A, base + S.scan[r], S.sortv[r] >> 12, S.acc[S.sortv[r] & 0xfff]);
  }
}

// ---- B5: bucket runs -> final order -------------------------------------------
// One warp per bucket (runs average tens of terms; a CTA per bucket left most
// of its threads idle).
__global__ void __launch_bounds__(256)
k_bucket_gather(const uint64_t* __restrict__ bbase, const uint32_t* __restrict__ bnnz,
                const uint64_t* __restrict__ boff, const uint64_t* __restrict__ sexp,
                const uint64_t* __restrict__ scoef, int nl, uint32_t nbuckets, uint64_t* __restrict__ oexp,
                uint64_t* __restrict__ ocoef) {
  const uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= nbuckets) return;
  const uint32_t n = bnnz[k];
  const uint64_t src = bbase[k], dst = boff[k];
  for (uint32_t t = lane; t < n; t += 32) oexp[dst + t] = sexp[src + t];
  for (uint32_t t = lane; t < n * (uint32_t)nl; t += 32) ocoef[dst * nl + t] = scoef[src * nl + t];
}

// bin offsets (exclusive scan of the fine-bin histogram)
struct BinOffOut {
  uint32_t* binoff;
  __device__ void operator()(uint64_t b, uint32_t ex, uint32_t) const { binoff[b] = ex; }
};
struct HistGen {
  const uint32_t* hist;
  __device__ uint32_t operator()(uint64_t b) const { return hist[b]; }
};

struct BnnzGen {
  const uint32_t* bnnz;
  __device__ uint64_t operator()(uint64_t k) const { return bnnz[k]; }
};
struct BoffOut {
  uint64_t* boff;
  __device__ void operator()(uint64_t k, uint64_t ex, uint64_t) const { boff[k] = ex; }
};

}  // namespace pgpu
