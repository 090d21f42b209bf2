// scan.cuh -- device-wide exclusive scan over a generated sequence.
//
// Reduce-then-scan over G contiguous block ranges: pass 1 sums each range,
// a single block scans the G partial sums, pass 2 rescans each range with its
// carry-in and hands (index, exclusive prefix, value) to an output functor.
// Each thread owns kScanIpt consecutive items of a tile (sequential inside the
// thread, one block scan per tile).  Used for row offsets, the sumset rank
// words, run-length heads and zero-coefficient compaction.
#pragma once
#include "common.cuh"

namespace pgpu {

constexpr int kScanThreads = 256;
constexpr int kScanIpt = 8;
constexpr int kScanTile = kScanThreads * kScanIpt;
constexpr int kMaxScanBlocks = 2048;

template <typename T, typename Gen>
__global__ void __launch_bounds__(kScanThreads)
k_range_reduce(uint64_t n, uint64_t per, Gen gen, T* part) {
  __shared__ T sh[33];
  const uint64_t beg = (uint64_t)blockIdx.x * per;
  const uint64_t end = beg + per < n ? beg + per : n;
  T s = 0;
  for (uint64_t i = beg + threadIdx.x; i < end; i += blockDim.x) s += gen(i);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    T v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : T(0);
    v = warp_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

// Exclusive scan of part[0..g) in place; part[g] = total.
template <typename T>
__global__ void __launch_bounds__(1024) k_part_scan(T* part, int g) {
  __shared__ T sh[33];
  T carry = 0;
  for (int base = 0; base < g; base += blockDim.x) {
    int i = base + threadIdx.x;
    T v = i < g ? part[i] : T(0);
    T tot;
    T ex = block_excl_scan(v, sh, &tot);
    if (i < g) part[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) part[g] = carry;
}

template <typename T, typename Gen, typename Out>
__global__ void __launch_bounds__(kScanThreads)
k_range_scan(uint64_t n, uint64_t per, Gen gen, Out out, const T* part) {
  __shared__ T sh[33];
  const uint64_t beg = (uint64_t)blockIdx.x * per;
  const uint64_t end = beg + per < n ? beg + per : n;
  T carry = part[blockIdx.x];
  for (uint64_t base = beg; base < end; base += kScanTile) {
    const uint64_t i0 = base + (uint64_t)threadIdx.x * kScanIpt;
    T v[kScanIpt];
    T s = 0;
#pragma unroll
    for (int k = 0; k < kScanIpt; ++k) {
      v[k] = (i0 + k < end) ? gen(i0 + k) : T(0);
      s += v[k];
    }
    T tot;
    T ex = block_excl_scan(s, sh, &tot) + carry;
#pragma unroll
    for (int k = 0; k < kScanIpt; ++k) {
      if (i0 + k < end) out(i0 + k, ex, v[k]);
      ex += v[k];
    }
    carry += tot;
  }
}

// Sum of gen(i) over [0, n) (the first two kernels of device_scan); the total
// lands in part[*g_out].  Returns the number of kernel launches (2).
template <typename T, typename Gen>
int device_sum(uint64_t n, Gen gen, T* part, int* g_out, cudaStream_t st) {
  uint64_t per = (uint64_t)kScanTile * 4;
  if ((n + per - 1) / per > (uint64_t)kMaxScanBlocks) per = (n + kMaxScanBlocks - 1) / kMaxScanBlocks;
  per = (per + kScanTile - 1) / kScanTile * kScanTile;
  int g = (int)((n + per - 1) / per);
  if (g < 1) g = 1;
  k_range_reduce<T><<<g, kScanThreads, 0, st>>>(n, per, gen, part);
  k_part_scan<T><<<1, 1024, 0, st>>>(part, g);
  *g_out = g;
  return 2;
}

constexpr unsigned long long kLbAgg = 1ull << 62;
constexpr unsigned long long kLbPre = 2ull << 62;
constexpr unsigned long long kLbVal = (1ull << 62) - 1;

// Decoupled look-back.  status[] is zeroed before the launch; a word holds a
// flag (kLbAgg / kLbPre) and a 62-bit value.  Tiles are claimed in order.
//
// tile_publish (one thread): tile k's count, as soon as it is known (tile 0:
// its inclusive prefix at once).
__device__ __forceinline__ void tile_publish(unsigned long long* status, uint32_t k, uint32_t agg) {
  *(volatile unsigned long long*)(status + k) = (k == 0 ? kLbPre : kLbAgg) | agg;
}

// tile_resolve (one whole warp): the exclusive prefix of the counts of tiles
// 0..k-1; with `finish`, lane 0 then publishes tile k's inclusive prefix.
// The warp reads 32 predecessors per round trip: it consumes the aggregates
// up to the nearest inclusive prefix, or up to the first predecessor not yet
// published (re-polled from there).  (Eight groups of 32 loads per round
// made the MP n=12 head scan 1.7x slower.)
__device__ __forceinline__ unsigned long long tile_resolve(unsigned long long* status, uint32_t k,
                                                           uint32_t agg, bool finish) {
  const int lane = threadIdx.x & 31;
  if (k == 0) return 0;
  unsigned long long excl = 0;
  int64_t q = (int64_t)k - 1;  // nearest predecessor not yet consumed
  for (;;) {
    const int64_t idx = q - lane;
    const unsigned long long v =
        idx >= 0 ? *(volatile unsigned long long*)(status + idx) : (unsigned long long)kLbPre;
    const unsigned long long flag = v & ~kLbVal;
    const unsigned pre = __ballot_sync(0xffffffffu, flag == kLbPre);
    const unsigned notready = __ballot_sync(0xffffffffu, flag == 0);
    const int first_pre = pre ? __ffs(pre) - 1 : 32;
    const unsigned upto = first_pre == 32 ? 0xffffffffu : ((2u << first_pre) - 1u);
    const unsigned wait = notready & upto;
    // lanes [0, take) are consumed: published aggregates, plus the prefix if no gap
    const int take = wait ? __ffs(wait) - 1 : (first_pre == 32 ? 32 : first_pre + 1);
    unsigned long long part = lane < take ? (v & kLbVal) : 0ull;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
    excl += part;
    q -= take;
    if (!wait && first_pre < 32) break;
  }
  if (finish && lane == 0) *(volatile unsigned long long*)(status + k) = kLbPre | (excl + agg);
  return excl;
}

// Both at once (one whole warp): publish, then resolve and finish.
__device__ __forceinline__ unsigned long long tile_lookback(unsigned long long* status, uint32_t k,
                                                            uint32_t agg) {
  if ((threadIdx.x & 31) == 0) tile_publish(status, k, agg);
  return tile_resolve(status, k, agg, true);
}

// ---- run heads (single pass) --------------------------------------------
// Runs of a sorted key array: equal keys (CONSEC = false: the sort path's
// segments) or consecutive keys k, k+1, k+2, ... (CONSEC = true: the dense
// path's operand runs).  One read of the keys: tiles of kHsTile keys are
// claimed in order (ticket), each thread flags the heads among its kHsIpt
// consecutive keys (16-byte loads), the block scans the flag counts, and warp
// 0 chains the tile totals by decoupled look-back.  Head r writes
// starts[r] = i and, when given, first[r] = keys[i] and last[r - 1] =
// keys[i - 1].  The last tile appends starts[nseg] = n (and last[nseg - 1])
// and stores nseg to *nseg_out.  status[] (ntiles words) and *ticket are
// zeroed before the launch.
#ifndef PGPU_HS_IPT
#define PGPU_HS_IPT 32
#endif
constexpr int kHsThreads = 256;
constexpr int kHsIpt = PGPU_HS_IPT;
constexpr int kHsTile = kHsThreads * kHsIpt;  // 32 keys per thread: MP n=12 heads 0.127 -> 0.095 ms
static_assert(kHsIpt <= 32, "head flags are one 32-bit mask per thread");

template <typename KT, bool CONSEC>
__global__ void __launch_bounds__(kHsThreads)
k_head_scan(const KT* __restrict__ keys, uint64_t n, uint32_t* __restrict__ starts,
            unsigned long long* __restrict__ status, uint32_t* __restrict__ ticket,
            uint32_t* __restrict__ nseg_out, KT* __restrict__ first = nullptr, KT* __restrict__ last = nullptr) {
  __shared__ uint32_t sh[33];
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t i0 = (uint64_t)tile * kHsTile + (uint64_t)threadIdx.x * kHsIpt;
  static_assert(sizeof(KT) * kHsIpt % 16 == 0, "whole 16-byte words per thread");
  constexpr int W = (int)(sizeof(KT) * kHsIpt / 16);
  union {
    uint4 w[W];
    KT k[kHsIpt];
  } u;
  KT prev = 0;  // key i0 - 1
  uint32_t m = 0;  // bit j: key i0+j is a head
  auto head = [](KT c, KT p) { return CONSEC ? c != (KT)(p + 1) : c != p; };
  if (i0 + kHsIpt <= n) {
    const uint4* src = reinterpret_cast<const uint4*>(keys + i0);
#pragma unroll
    for (int j = 0; j < W; ++j) u.w[j] = __ldg(src + j);
    prev = i0 ? keys[i0 - 1] : (KT)0;
    KT p = prev;
#pragma unroll
    for (int j = 0; j < kHsIpt; ++j) {
      m |= (i0 + j == 0 || head(u.k[j], p) ? 1u : 0u) << j;
      p = u.k[j];
    }
  } else if (i0 < n) {
    prev = i0 ? keys[i0 - 1] : (KT)0;
    KT p = prev;
    for (int j = 0; j < kHsIpt && i0 + j < n; ++j) {
      u.k[j] = keys[i0 + j];
      m |= (i0 + j == 0 || head(u.k[j], p) ? 1u : 0u) << j;
      p = u.k[j];
    }
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan((uint32_t)__popc(m), sh, &tot);
  if (threadIdx.x < 32) {
    const unsigned long long e = tile_lookback(status, tile, tot);
    if (threadIdx.x == 0) s_excl = e;
  }
  __syncthreads();
  ex += (uint32_t)s_excl;
  while (m) {
    const int j = __ffs(m) - 1;
    m &= m - 1;
    starts[ex] = (uint32_t)(i0 + j);
    if (first) first[ex] = u.k[j];
    if (last && ex > 0) last[ex - 1] = j ? u.k[j - 1] : prev;
    ++ex;
  }
  const uint64_t ntiles = (n + kHsTile - 1) / kHsTile;
  if (threadIdx.x == 0 && tile == ntiles - 1) {
    const uint32_t nseg = (uint32_t)s_excl + tot;
    starts[nseg] = (uint32_t)n;
    if (last) last[nseg - 1] = keys[n - 1];
    *nseg_out = nseg;
  }
}

// Host driver.  `part` must hold >= kMaxScanBlocks+1 elements.
// Returns the number of kernel launches (3).  The total lands in part[*g_out].
template <typename T, typename Gen, typename Out>
int device_scan(uint64_t n, Gen gen, Out out, T* part, int* g_out, cudaStream_t st) {
  // ~4 tiles per block, at most kMaxScanBlocks blocks
  uint64_t per = (uint64_t)kScanTile * 4;
  if ((n + per - 1) / per > (uint64_t)kMaxScanBlocks) per = (n + kMaxScanBlocks - 1) / kMaxScanBlocks;
  per = (per + kScanTile - 1) / kScanTile * kScanTile;
  int g = (int)((n + per - 1) / per);
  if (g < 1) g = 1;
  k_range_reduce<T><<<g, kScanThreads, 0, st>>>(n, per, gen, part);
  k_part_scan<T><<<1, 1024, 0, st>>>(part, g);
  k_range_scan<T><<<g, kScanThreads, 0, st>>>(n, per, gen, out, part);
  *g_out = g;
  return 3;
}

}  // namespace pgpu
