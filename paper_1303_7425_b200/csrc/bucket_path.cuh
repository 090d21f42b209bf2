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
//   B4 k_bucket_reduce persistent CTAs claim buckets in key order: each
//                     distinct key ranked (a bitmap over the bucket's key
//                     span with a popcount prefix per word; a shared-memory
//                     hash for buckets spanning more than kBkWords*32 keys),
//                     records placed in (key, row)
//                     order, products folded by one owner per key in that
//                     order (no atomics on coefficient data: integers exact,
//                     doubles in the reference's order and run-to-run
//                     identical), zero sums dropped (merge.py:63); terms go
//                     to their final positions: the CTA's previous bucket's
//                     inclusive prefix plus the published term counts of the
//                     buckets claimed in between.  A bin above the bucket bound
//                     sends the batch to the sort path.
//
// DRAM traffic per pair: one record write + one record read (12-16 B each),
// against 5-6 read+write passes on the sort path.
#pragma once
#include "common.cuh"
#include "scan.cuh"

namespace pgpu {

#ifndef PGPU_BUCKET_CAP
#define PGPU_BUCKET_CAP 2048
#endif
constexpr int kBucketCap = PGPU_BUCKET_CAP;  // pairs per bucket (max)
constexpr int kBucketHalf = kBucketCap / 2;
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
              uint32_t* __restrict__ fill, KT* __restrict__ rkey, uint64_t* __restrict__ rid,
              uint64_t cap) {
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
      PGPU_ASSERT(!valid || pos < cap);
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
// Persistent CTAs claim buckets in key order.  A bucket's records are grouped
// by key without touching coefficient data atomically:
//   1-3. every record gets its key's rank among the bucket's distinct keys.
//      Bitmap (keys spanning <= kBkWords*32 values, the common case): one
//      shared-memory atomicOr per record sets bit key - lo, a block scan of
//      the words' popcounts gives each word's rank base, and a record's rank
//      is base + popc(word & bits below its key): no comparisons.  Hash
//      (wider spans): keys -> open-addressing slots (CAS on the key only),
//      distinct keys compacted and ranked (counting rank, or a bitonic sort
//      above 224).  The distinct-key count is published at once (successors
//      need it for their output base)
//   4. per key rank: record count (the returned index is an arbitrary position
//      in the key's run), exclusive scan -> run starts; each record's position
//      in (key, row) order: floats rank their row among the run's rows (the
//      reference's tie order, merge.py:32-33), integers keep the arbitrary
//      position (exact sums do not depend on the order)
//   5. each record's product is written at its position; warp 0 then resolves
//      the bucket's output base (bucket_base: this CTA's previous inclusive
//      prefix + the counts of the buckets claimed in between, one round of
//      loads instead of a look-back walk over buckets in flight)
//   6. one owner per key folds its run in order (acc = p_first; acc += p ...;
//      merge.py:49-58) and writes term base + rank: no staging and no gather
//      pass.  A zero sum (merge.py:63) leaves its slot marked with the
//      all-ones exponent (SENTINEL, never a term) and is counted; the driver
//      compacts only if any occurred.
constexpr int kBkIpt = kBucketCap / kBucketThreads;  // records per thread
constexpr int kBkTable = 2 * kBucketCap;             // hash slots (load factor <= 1/2)
constexpr int kBkSlotBits = 12;
static_assert(kBkTable <= (1 << kBkSlotBits), "slot index must fit the sort word");
constexpr uint32_t kBkRankThreads = kBucketThreads - 32;  // warp 0 runs the look-back meanwhile

struct BucketArgs {
  const void* rkey;            // KT keys relative to KL
  const uint64_t* rid;         // i<<32 | j
  const uint32_t* binoff;      // nbins offsets
  const uint32_t* bstart;      // nbuckets+1 first bins
  uint32_t nbins, pairs, nbuckets;
  const void* ac;
  const void* bc;
  uint64_t KL;
  KeyPlan P;
  uint64_t* oexp;              // distinct keys in key order (capacity: pairs)
  uint64_t* ocoef;             // NL limbs per term (f64: the double's bits)
  unsigned long long* status;  // [nbuckets] look-back words (zeroed)
  unsigned int* ticket;        // next bucket to claim (zeroed)
  uint32_t* overflow;          // a bucket above kBucketCap records: the batch takes the sort path
  unsigned long long* zeros;   // zero sums written as holes
};

// Buckets whose keys span at most kBkWords*32 values rank them with a bitmap
// (one bit per key of the span, popcount prefix per word); wider ones hash.
#ifndef PGPU_BK_WORDS
#define PGPU_BK_WORDS (PGPU_BUCKET_CAP >= 2048 ? 2048 : 1024)
#endif
constexpr int kBkWords = PGPU_BK_WORDS;
static_assert(kBkWords % kBucketThreads == 0, "whole words per thread");

template <typename KT, int NL, bool ROWS>
struct BucketSmem {
  union {
    struct {
      KT hkey[kBkTable];             // open-addressing key table
      uint16_t rank[kBkTable];       // key rank of an occupied slot
    } h;
    struct {
      uint32_t bits[kBkWords];       // key k - lo present: bit (k - lo) & 31 of word (k - lo) >> 5
      uint16_t wpre[kBkWords];       // distinct keys before the word
    } m;
  };
  union {
    uint64_t sortv[kBucketCap];      // distinct keys: key << 12 | slot
    uint64_t prod[kBucketCap * NL];  // products at their (key, row) positions; then run sums
  };
  KT keyr[kBucketCap];               // key of each rank
  uint32_t start[kBucketCap + 1];    // per key rank: count, then run start
  uint32_t rows[ROWS ? kBucketCap : 1];  // rows at arbitrary run positions (f64 tie order)
  uint32_t sh[33];
  KT kext[2][kBucketThreads / 32];   // per-warp key minimum / maximum
  uint32_t bucket;
  unsigned long long base;
};

__device__ __forceinline__ uint32_t cas_key(uint32_t* p, uint32_t cmp, uint32_t v) {
  return atomicCAS(reinterpret_cast<unsigned int*>(p), cmp, v);
}
__device__ __forceinline__ uint64_t cas_key(uint64_t* p, uint64_t cmp, uint64_t v) {
  return atomicCAS(reinterpret_cast<unsigned long long*>(p), (unsigned long long)cmp,
                   (unsigned long long)v);
}

// Bucket status words (zeroed before the launch): bit 63 = the bucket's term
// count is published (bits 0-15); bit 62 = its inclusive prefix too (bits
// 16-61, read by the host for the last bucket).
constexpr unsigned long long kBsCnt = 1ull << 63;
constexpr unsigned long long kBsIncl = 1ull << 62;

__device__ __forceinline__ void bucket_publish(unsigned long long* status, uint32_t k, uint32_t nd) {
  *(volatile unsigned long long*)(status + k) = kBsCnt | nd;
}

// Output base of bucket k (one whole warp).  Every CTA knows the inclusive
// prefix of its own previous bucket kp (kp = -1: prefix 0), so the base is
// that prefix plus the counts of the buckets claimed in between -- published
// as soon as each bucket has ranked its keys.  The warp loads them all at once
// (16 per lane per round, ~one bucket per resident CTA in between): one L2
// round trip instead of a look-back walk over buckets still in flight.
__device__ __forceinline__ unsigned long long bucket_base(const unsigned long long* status, uint32_t k,
                                                          int64_t kp, unsigned long long pre) {
  constexpr int U = 16;
  const int lane = threadIdx.x & 31;
  unsigned long long sum = 0;
  for (int64_t j0 = kp + 1; j0 < (int64_t)k; j0 += 32 * U) {
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + lane + 32 * u;
      v[u] = j < (int64_t)k ? *(const volatile unsigned long long*)(status + j) : kBsCnt;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + lane + 32 * u;
      while (!(v[u] & kBsCnt)) v[u] = *(const volatile unsigned long long*)(status + j);
      sum += v[u] & 0xffffull;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
  return pre + sum;
}

__device__ __forceinline__ uint32_t warp_min_key(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint32_t warp_max_key(uint32_t v) { return __reduce_max_sync(0xffffffffu, v); }
__device__ __forceinline__ uint64_t warp_min_key(uint64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t o = __shfl_xor_sync(0xffffffffu, v, d);
    v = o < v ? o : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_max_key(uint64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t o = __shfl_xor_sync(0xffffffffu, v, d);
    v = o > v ? o : v;
  }
  return v;
}

__device__ __forceinline__ uint32_t bucket_hash(uint64_t k) {
  return (uint32_t)((k * 0x9E3779B97F4A7C15ull) >> 40) & (kBkTable - 1);
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

// ---- block bitonic sort of 256*E words held blocked (thread t: [t*E, t*E+E)) --
__device__ __forceinline__ void bitonic_keep(uint64_t& a, uint64_t o, uint32_t x, uint32_t s, uint32_t k) {
  const bool up = (x & k) == 0, lower = (x & s) == 0;
  const uint64_t lo = a < o ? a : o, hi = a < o ? o : a;
  a = (lower == up) ? lo : hi;
}

template <int E, int S>
__device__ __forceinline__ void bitonic_reg(uint64_t (&v)[E], uint32_t t, uint32_t k) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if ((e & S) == 0) {
      const bool up = ((t * E + e) & k) == 0;
      const uint64_t a = v[e], b = v[e + S];
      if ((a > b) == up) {
        v[e] = b;
        v[e + S] = a;
      }
    }
  }
}

// strides below E inside a thread, below 32E across lanes (shuffles), larger
// ones through `xch` (>= 256*E words of shared memory)
template <int E>
__device__ void block_bitonic(uint64_t (&v)[E], uint64_t* xch) {
  constexpr uint32_t N = kBucketThreads * E;
  const uint32_t t = threadIdx.x;
#pragma unroll 1
  for (uint32_t k = 2; k <= N; k <<= 1) {
#pragma unroll 1
    for (uint32_t s = k >> 1; s > 0; s >>= 1) {
      if (s >= 32u * E) {
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) xch[t * E + e] = v[e];
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) bitonic_keep(v[e], xch[(t * E + e) ^ s], t * E + e, s, k);
      } else if (s >= (uint32_t)E) {
        const int ld = (int)(s / E);
#pragma unroll
        for (int e = 0; e < E; ++e)
          bitonic_keep(v[e], __shfl_xor_sync(0xffffffffu, v[e], ld), t * E + e, s, k);
      } else {
        if constexpr (E >= 8) {
          if (s == 4) bitonic_reg<E, 4>(v, t, k);
        }
        if constexpr (E >= 4) {
          if (s == 2) bitonic_reg<E, 2>(v, t, k);
        }
        if constexpr (E >= 2) {
          if (s == 1) bitonic_reg<E, 1>(v, t, k);
        }
      }
    }
  }
  __syncthreads();
}

// key rank of every occupied slot: rank[slot] and keyr[rank]
template <typename KT, int NL, bool ROWS, int E>
__device__ __forceinline__ void rank_sorted(BucketSmem<KT, NL, ROWS>& S, uint32_t nd) {
  uint64_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t x = threadIdx.x * E + e;
    v[e] = x < nd ? S.sortv[x] : ~0ull;
  }
  block_bitonic<E>(v, S.sortv);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t x = threadIdx.x * E + e;
    if (x < nd) {
      S.h.rank[v[e] & ((1u << kBkSlotBits) - 1)] = (uint16_t)x;
      S.keyr[x] = (KT)(v[e] >> kBkSlotBits);
    }
  }
}

// counting rank (threads 32.., C keys each): the number of smaller distinct keys
template <typename KT, int NL, bool ROWS, int C>
__device__ __forceinline__ void rank_counting(BucketSmem<KT, NL, ROWS>& S, uint32_t nd) {
  const uint32_t t = threadIdx.x - 32;
  KT mine[C];
  uint32_t rk[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const uint32_t x = t + c * kBkRankThreads;
    mine[c] = x < nd ? (KT)(S.sortv[x] >> kBkSlotBits) : (KT)~(KT)0;
    rk[c] = 0;
  }
  // the keys, narrowed to KT, were stored in keyr[] in slot order by the caller
  if constexpr (sizeof(KT) == 4) {
    // o < mine <=> o - mine borrows: two instructions per comparison
    uint32_t neg[C];
#pragma unroll
    for (int c = 0; c < C; ++c) neg[c] = 0;
#pragma unroll 4
    for (uint32_t y = 0; y < nd; ++y) {
      const uint32_t o = (uint32_t)S.keyr[y];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        uint32_t tmp;
        asm("sub.cc.u32 %0, %2, %3;\n\tsubc.u32 %1, %1, 0;" : "=r"(tmp), "+r"(neg[c]) : "r"(o), "r"((uint32_t)mine[c]));
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) rk[c] = 0u - neg[c];
  } else {
    for (uint32_t y = 0; y < nd; ++y) {
      const KT o = S.keyr[y];
#pragma unroll
      for (int c = 0; c < C; ++c) rk[c] += o < mine[c] ? 1u : 0u;
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const uint32_t x = t + c * kBkRankThreads;
    if (x < nd) S.h.rank[S.sortv[x] & ((1u << kBkSlotBits) - 1)] = (uint16_t)rk[c];
  }
}

// CK: 0 f64, 1 int64, 2 int128 operands; NL result limbs
#ifndef PGPU_BUCKET_MINB
#define PGPU_BUCKET_MINB (768 / PGPU_BUCKET_THREADS)
#endif
template <typename KT, int NL, int CK>
__global__ void __launch_bounds__(kBucketThreads, NL <= 2 ? PGPU_BUCKET_MINB : (PGPU_BUCKET_MINB * 2 + 2) / 3)
k_bucket_reduce(BucketArgs A) {
  constexpr bool ROWS = CK == 0;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  BucketSmem<KT, NL, ROWS>& S = *reinterpret_cast<BucketSmem<KT, NL, ROWS>*>(smem_raw);
  const KT kEmpty = (KT)~(KT)0;
  int64_t kp = -1;             // this CTA's previous bucket
  unsigned long long pre = 0;  // and its inclusive term prefix
  for (;;) {
    __syncthreads();  // the previous bucket's readers are done with the shared state
    if (threadIdx.x == 0) S.bucket = atomicAdd(A.ticket, 1u);
    // the key bitmap starts clear (the common case; the hash table is set up
    // only by the buckets that need it)
#pragma unroll
    for (int u = 0; u < kBkWords / (4 * kBucketThreads); ++u)
      reinterpret_cast<uint4*>(S.m.bits)[threadIdx.x + u * kBucketThreads] = make_uint4(0, 0, 0, 0);
    for (uint32_t x = threadIdx.x; x <= (uint32_t)kBucketCap; x += kBucketThreads) S.start[x] = 0;
    __syncthreads();
    const uint32_t k = S.bucket;
    if (k >= A.nbuckets) return;
    const uint32_t b0 = A.bstart[k], b1 = A.bstart[k + 1];
    const uint32_t r0 = A.binoff[b0];
    const uint32_t r1 = b1 < A.nbins ? A.binoff[b1] : A.pairs;
    const uint32_t n = r1 - r0;
    if (n > (uint32_t)kBucketCap) {  // one fine bin above the bucket bound
      if (threadIdx.x == 0) {
        *A.overflow = 1u;
        bucket_publish(A.status, k, 0);
      }
      continue;
    }
    // records (coalesced) and the bucket's key extent
    uint64_t id[kBkIpt];
    uint32_t slot[kBkIpt];  // the record's key rank after step 3
    uint32_t valid = 0;
    KT key[kBkIpt];
    {
      const KT* __restrict__ rkey = reinterpret_cast<const KT*>(A.rkey) + r0;
      const uint64_t* __restrict__ rid = A.rid + r0;
      KT lmin = kEmpty, lmax = 0;
#pragma unroll
      for (int u = 0; u < kBkIpt; ++u) {
        const uint32_t q = threadIdx.x + u * kBucketThreads;
        key[u] = q < n ? rkey[q] : kEmpty;
        id[u] = q < n ? rid[q] : 0ull;
        valid |= (q < n ? 1u : 0u) << u;
        if (q < n) {
          lmin = key[u] < lmin ? key[u] : lmin;
          lmax = key[u] > lmax ? key[u] : lmax;
        }
      }
      lmin = warp_min_key(lmin);
      lmax = warp_max_key(lmax);
      if ((threadIdx.x & 31) == 0) {
        S.kext[0][threadIdx.x >> 5] = lmin;
        S.kext[1][threadIdx.x >> 5] = lmax;
      }
    }
    __syncthreads();
    KT kmin = S.kext[0][0], kmax = S.kext[1][0];
#pragma unroll
    for (int q = 1; q < kBucketThreads / 32; ++q) {
      kmin = S.kext[0][q] < kmin ? S.kext[0][q] : kmin;
      kmax = S.kext[1][q] > kmax ? S.kext[1][q] : kmax;
    }
    const KT lo = kmin & ~(KT)31;
    uint32_t nd;
    if (n == 0 || (uint64_t)(kmax - lo) < 32ull * kBkWords) {
      // 1-3 (bitmap): mark each key's bit; a key's rank is the number of marked
      // bits before it (popcount prefix per word); no comparisons
#pragma unroll
      for (int u = 0; u < kBkIpt; ++u)
        if ((valid >> u) & 1u) {
          const uint32_t off = (uint32_t)(key[u] - lo);
          atomicOr(&S.m.bits[off >> 5], 1u << (off & 31));
        }
      __syncthreads();
      constexpr int WPT = kBkWords / kBucketThreads;  // consecutive words per thread
      static_assert(WPT % 8 == 0 || WPT == 4, "whole 16-byte loads and stores per thread");
      uint32_t c[WPT];
      {
        const uint4* bw = reinterpret_cast<const uint4*>(S.m.bits) + (WPT / 4) * threadIdx.x;
#pragma unroll
        for (int q = 0; q < WPT / 4; ++q) {
          const uint4 x = bw[q];
          c[4 * q] = __popc(x.x);
          c[4 * q + 1] = __popc(x.y);
          c[4 * q + 2] = __popc(x.z);
          c[4 * q + 3] = __popc(x.w);
        }
      }
      uint32_t cnt = 0;
#pragma unroll
      for (int q = 0; q < WPT; ++q) cnt += c[q];
      uint32_t ex = block_excl_scan(cnt, S.sh, &nd);
      uint32_t pw[WPT / 2];
#pragma unroll
      for (int q = 0; q < WPT; q += 2) {
        pw[q / 2] = ex | ((ex + c[q]) << 16);
        ex += c[q] + c[q + 1];
      }
      if constexpr (WPT == 4) {
        reinterpret_cast<uint2*>(S.m.wpre)[threadIdx.x] = make_uint2(pw[0], pw[1]);
      } else {
#pragma unroll
        for (int q = 0; q < WPT / 8; ++q)
          reinterpret_cast<uint4*>(S.m.wpre)[(WPT / 8) * threadIdx.x + q] =
              make_uint4(pw[4 * q], pw[4 * q + 1], pw[4 * q + 2], pw[4 * q + 3]);
      }
      __syncthreads();
      // the bucket's term count goes out now (its successors' bases need it)
      if (threadIdx.x == 0) bucket_publish(A.status, k, nd);
#pragma unroll
      for (int u = 0; u < kBkIpt; ++u)
        if ((valid >> u) & 1u) {
          const uint32_t off = (uint32_t)(key[u] - lo);
          const uint32_t wd = off >> 5;
          slot[u] = S.m.wpre[wd] + __popc(S.m.bits[wd] & ((1u << (off & 31)) - 1u));
          S.keyr[slot[u]] = key[u];  // (every record of the key writes the same value)
        }
    } else {
      // 1. slot per distinct key (open addressing, CAS on the key only)
#pragma unroll
      for (int u = 0; u < kBkTable / kBucketThreads; ++u) S.h.hkey[threadIdx.x + u * kBucketThreads] = kEmpty;
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kBkIpt; ++u) {
        uint32_t h = 0;
        if ((valid >> u) & 1u) {
          h = bucket_hash((uint64_t)key[u]);
          for (;;) {
            const KT prev = cas_key(&S.h.hkey[h], kEmpty, key[u]);
            if (prev == kEmpty || prev == key[u]) break;
            h = (h + 1) & (kBkTable - 1);
          }
        }
        slot[u] = h;
      }
      __syncthreads();
      // 2. distinct keys compacted in slot order (thread t scans slots [16t, 16t+16))
      constexpr int TPT = kBkTable / kBucketThreads;
      {
        const uint32_t t0 = threadIdx.x * TPT;
        uint32_t occ = 0, cnt = 0;
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
          const bool o = S.h.hkey[t0 + u] != kEmpty;
          occ |= (o ? 1u : 0u) << u;
          cnt += o ? 1u : 0u;
        }
        uint32_t at = block_excl_scan(cnt, S.sh, &nd);
#pragma unroll
        for (int u = 0; u < TPT; ++u) {
          if ((occ >> u) & 1u) {
            const KT kk = S.h.hkey[t0 + u];
            S.sortv[at] = ((uint64_t)kk << kBkSlotBits) | (t0 + u);
            S.keyr[at] = kk;  // slot order (counting rank input); rank order after step 3
            ++at;
          }
        }
      }
      __syncthreads();
      // 3. the term count goes out (warp 0) while the other warps rank the keys
      if (nd <= 2u * kBkRankThreads) {
        if (threadIdx.x < 32) {
          if (threadIdx.x == 0) bucket_publish(A.status, k, nd);
        } else if (nd <= kBkRankThreads) {
          rank_counting<KT, NL, ROWS, 1>(S, nd);
        } else {
          rank_counting<KT, NL, ROWS, 2>(S, nd);
        }
        __syncthreads();
        // keys in rank order (keyr held them in slot order for the counting rank)
        constexpr int RC = (2 * kBkRankThreads + kBucketThreads - 1) / kBucketThreads;
        KT kk[RC];
        uint32_t rk[RC];
#pragma unroll
        for (int c = 0; c < RC; ++c) {
          const uint32_t x = threadIdx.x + c * kBucketThreads;
          if (x < nd) {
            kk[c] = S.keyr[x];
            rk[c] = S.h.rank[S.sortv[x] & ((1u << kBkSlotBits) - 1)];
          }
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < RC; ++c)
          if (threadIdx.x + c * kBucketThreads < nd) S.keyr[rk[c]] = kk[c];
      } else {
        if (threadIdx.x == 0) bucket_publish(A.status, k, nd);
        if (nd <= 4u * kBucketThreads) rank_sorted<KT, NL, ROWS, 4>(S, nd);
        else rank_sorted<KT, NL, ROWS, 8>(S, nd);
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kBkIpt; ++u)
        if ((valid >> u) & 1u) slot[u] = S.h.rank[slot[u]];  // slot -> key rank
    }
    __syncthreads();
    // 4. runs: count per key rank (the index is an arbitrary position in the run)
    uint32_t pos[kBkIpt];
#pragma unroll
    for (int u = 0; u < kBkIpt; ++u)
      if ((valid >> u) & 1u) pos[u] = atomicAdd(&S.start[slot[u]], 1u);
    if (threadIdx.x == 0) S.start[nd] = n;
    __syncthreads();
    chunk_scan<kBkIpt>(S.start, nd, S.sh);
    // position in (key, row) order
    if constexpr (ROWS) {
#pragma unroll
      for (int u = 0; u < kBkIpt; ++u)
        if ((valid >> u) & 1u) {
          PGPU_ASSERT(slot[u] < nd && S.start[slot[u]] + pos[u] < S.start[slot[u] + 1]);
          S.rows[S.start[slot[u]] + pos[u]] = (uint32_t)(id[u] >> 32);
        }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kBkIpt; ++u) {
        if ((valid >> u) & 1u) {
          const uint32_t s0 = S.start[slot[u]], len = S.start[slot[u] + 1] - s0;
          const uint32_t i = (uint32_t)(id[u] >> 32);
          uint32_t below = 0;
          for (uint32_t x = 0; x < len; ++x) below += S.rows[s0 + x] < i ? 1u : 0u;
          pos[u] = s0 + below;
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < kBkIpt; ++u)
        if ((valid >> u) & 1u) pos[u] += S.start[slot[u]];
    }
    // 5. products at their positions (sortv is dead: the ranks are in rank[]/keyr[])
#pragma unroll
    for (int u = 0; u < kBkIpt; ++u) {
      if (!((valid >> u) & 1u)) continue;
      PGPU_ASSERT(slot[u] < nd && pos[u] >= S.start[slot[u]] && pos[u] < S.start[slot[u] + 1] && pos[u] < n);
      const uint64_t i = id[u] >> 32, j = id[u] & 0xffffffffu;
      if constexpr (CK == 0) {
        const double pr = __dmul_rn(__ldg(reinterpret_cast<const double*>(A.ac) + i),
                                    __ldg(reinterpret_cast<const double*>(A.bc) + j));
        S.prod[pos[u]] = (uint64_t)__double_as_longlong(pr);
      } else {
        const Limbs<NL> pr = imul<NL, CK>(load_icoef<CK>(A.ac, (int64_t)i), load_icoef<CK>(A.bc, (int64_t)j));
#pragma unroll
        for (int w = 0; w < NL; ++w) S.prod[(size_t)pos[u] * NL + w] = pr.w[w];
      }
    }
    // output base (warp 0, after its products; the barrier below waits for it)
    if (threadIdx.x < 32) {
      const unsigned long long b = bucket_base(A.status, k, kp, pre);
      if (threadIdx.x == 0) {
        S.base = b;
        *(volatile unsigned long long*)(A.status + k) = kBsCnt | kBsIncl | ((b + nd) << 16) | nd;
      }
    }
    __syncthreads();
    // 6. one owner per key folds its run in order and writes term base + rank
    const unsigned long long base = S.base;
    kp = k;
    pre = base + nd;
    uint32_t nzero = 0;
    for (uint32_t r = threadIdx.x; r < nd; r += kBucketThreads) {
      const uint32_t s0 = S.start[r], s1 = S.start[r + 1];
      bool nz;
      uint64_t out[NL];
      if constexpr (CK == 0) {
        double acc = __longlong_as_double((long long)S.prod[s0]);
        for (uint32_t x = s0 + 1; x < s1; ++x) acc = __dadd_rn(acc, __longlong_as_double((long long)S.prod[x]));
        out[0] = (uint64_t)__double_as_longlong(acc);
        nz = acc != 0.0;  // NaN kept, +-0 dropped (merge.py:63)
      } else {
        Limbs<NL> acc;
#pragma unroll
        for (int w = 0; w < NL; ++w) acc.w[w] = S.prod[(size_t)s0 * NL + w];
        for (uint32_t x = s0 + 1; x < s1; ++x) {
          Limbs<NL> p;
#pragma unroll
          for (int w = 0; w < NL; ++w) p.w[w] = S.prod[(size_t)x * NL + w];
          limbs_add(acc, p);
        }
#pragma unroll
        for (int w = 0; w < NL; ++w) out[w] = acc.w[w];
        nz = limbs_nonzero(acc);
      }
      const uint64_t o = base + r;
      PGPU_ASSERT(o < A.pairs && s0 < s1 && s1 <= n);
      A.oexp[o] = nz ? expand_key(A.KL + (uint64_t)S.keyr[r], A.P) : ~0ull;
#pragma unroll
      for (int w = 0; w < NL; ++w) A.ocoef[o * NL + w] = out[w];
      nzero += nz ? 0u : 1u;
    }
    if (nzero) atomicAdd(A.zeros, (unsigned long long)nzero);
  }
}

// terms present (not a zero-sum hole marked by the all-ones exponent)
struct HoleGen {
  const uint64_t* exps;
  __device__ uint32_t operator()(uint64_t i) const { return exps[i] != ~0ull ? 1u : 0u; }
};

// bin offsets (exclusive scan of the fine-bin histogram)
struct BinOffOut {
  uint32_t* binoff;
  __device__ void operator()(uint64_t b, uint32_t ex, uint32_t) const { binoff[b] = ex; }
};
struct HistGen {
  const uint32_t* hist;
  __device__ uint32_t operator()(uint64_t b) const { return hist[b]; }
};

}  // namespace pgpu
