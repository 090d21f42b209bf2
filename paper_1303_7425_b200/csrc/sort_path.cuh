// sort_path.cuh -- the general "expand / sort / run-length reduce" pipeline.
//
// This is the north star's materialise-sort-reduce design and the path taken
// for any input (wide keys, sparse products, the bit-exact float mode):
//
//   K1 k_gen        every pair (i, j) of a key range -> (compact key, i<<32|j)
//                   (replaces the (a_i+b_j, i, j) creation of merge.py:41-60)
//   K2 radix sort   stable LSD, 8-bit digits, on the significant key bits only
//                   (replaces heapq ordering, merge.py:42-62; stability keeps
//                   equal keys in increasing i, the reference's tie order)
//   K3 heads/scan   run-length heads where the key changes -> segment starts
//                   (replaces equal-exponent combining, merge.py:54-62)
//   K4 seg reduce   one thread owns one output term and folds its segment in
//                   order (acc = p_first; acc += p ...), merge.py:49-58
//   K5 nz compact   drop zero sums (merge.py:63)
//
// Products of 2^20 pairs or more use 8-byte records (local key, column j):
// k_gen_j writes them, K4 recovers each pair's row from its key through a
// hash of operand a's keys (k_seg_reduce_*_j).
#pragma once
#include <type_traits>
#include "common.cuh"
#include "scan.cuh"

namespace pgpu {

// ---- K1: pair generation ---------------------------------------------------
// One warp per row, lanes over consecutive columns: coalesced key loads and
// coalesced record stores.  Row i's pairs land at off[i] in increasing j, rows
// in increasing i, so the generation order is the reference's (i, j) order.
// KT: operand compact keys; RT: record keys (key - KL), u32 when the batch's
// key span fits 32 bits even if the operands' keys do not.
template <typename KT, typename RT>
__global__ void __launch_bounds__(256)
k_gen(const KT* __restrict__ ak, const KT* __restrict__ bk, const uint32_t* __restrict__ rlo,
      const uint32_t* __restrict__ rhi, const uint64_t* __restrict__ off, uint32_t na,
      uint64_t KL, RT* __restrict__ keys, uint64_t* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < na; i += nwarps) {
    uint32_t j0 = rlo[i], j1 = rhi[i];
    if (j0 >= j1) continue;
    uint64_t base = off[i] - j0;
    uint64_t ai = (uint64_t)ak[i] - KL;  // wraps for rows below KL; the sum does not
    for (uint32_t j = j0 + lane; j < j1; j += 32) {
      keys[base + j] = (RT)(ai + (uint64_t)__ldg(bk + j));
      vals[base + j] = ((uint64_t)i << 32) | j;
    }
  }
}

// K1 with 32-bit records: the value is the column j only.  The row is
// recovered in K4 from the key: a_i = key + KL - b_j, looked up in a hash of
// the operand a keys (keys of a are distinct).  12 -> 8 bytes per record
// through every radix pass.
template <typename KT, typename RT>
__global__ void __launch_bounds__(256)
k_gen_j(const KT* __restrict__ ak, const KT* __restrict__ bk, const uint32_t* __restrict__ rlo,
        const uint32_t* __restrict__ rhi, const uint64_t* __restrict__ off, uint32_t na,
        uint64_t KL, RT* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < na; i += nwarps) {
    uint32_t j0 = rlo[i], j1 = rhi[i];
    if (j0 >= j1) continue;
    uint64_t base = off[i] - j0;
    uint64_t ai = (uint64_t)ak[i] - KL;
    for (uint32_t j = j0 + lane; j < j1; j += 32) {
      keys[base + j] = (RT)(ai + (uint64_t)__ldg(bk + j));
      vals[base + j] = j;
    }
  }
}

__device__ __forceinline__ uint32_t row_hash(uint64_t k) {
  return (uint32_t)((k * 0x9E3779B97F4A7C15ull) >> 32);
}

// A key and its operand coefficient in one 32-byte slot, so the segment
// reduce gathers one sector per operand term instead of a key, a row index
// and a coefficient from three arrays (MP n=25: 4 -> 2 sectors per pair).
// c0/c1: f64 bits in c0; int64 in c0 (c1 its sign); int128 limbs.
struct alignas(32) KCSlot {
  uint64_t key;  // all-ones: empty (hash of operand a)
  uint64_t c0, c1, pad;
};

template <int CK>
__device__ __forceinline__ void kc_set_coef(KCSlot& s, const void* coef, uint32_t i) {
  if constexpr (CK == 2) {
    s.c0 = reinterpret_cast<const uint64_t*>(coef)[2 * (uint64_t)i];
    s.c1 = reinterpret_cast<const uint64_t*>(coef)[2 * (uint64_t)i + 1];
  } else {
    s.c0 = reinterpret_cast<const uint64_t*>(coef)[i];
    s.c1 = (uint64_t)((int64_t)s.c0 >> 63);
  }
}

// operand b as slots: brec[j] = {bk[j], bc[j]}
template <typename KT, int CK>
__global__ void __launch_bounds__(256)
k_kc_fill(const KT* __restrict__ bk, const void* __restrict__ bc, uint32_t nb, KCSlot* __restrict__ brec) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nb) return;
  KCSlot s;
  s.key = (uint64_t)bk[j];
  kc_set_coef<CK>(s, bc, j);
  s.pad = 0;
  brec[j] = s;
}

// open-addressing table key -> (key, coefficient) of operand a (keys of a
// are distinct; slots pre-filled with all-ones keys)
template <typename KT, int CK>
__global__ void __launch_bounds__(256)
k_kc_hash_build(const KT* __restrict__ ak, const void* __restrict__ ac, uint32_t na, KCSlot* __restrict__ slots,
                uint32_t mask) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= na) return;
  const uint64_t key = (uint64_t)ak[i];
  uint32_t h = row_hash(key) & mask;
  for (;;) {
    const unsigned long long prev =
        atomicCAS(reinterpret_cast<unsigned long long*>(&slots[h].key), ~0ull, (unsigned long long)key);
    if (prev == ~0ull) {
      kc_set_coef<CK>(slots[h], ac, i);
      return;
    }
    h = (h + 1) & mask;
  }
}

struct KCHash {
  const KCSlot* slots;
  uint32_t mask;
  __device__ __forceinline__ KCSlot find(uint64_t key) const {
    uint32_t h = row_hash(key) & mask;
    for (;;) {
      const KCSlot e = slots[h];
      if (e.key == key) return e;
      h = (h + 1) & mask;
    }
  }
};

template <int CK>
__device__ __forceinline__ ICoef kc_icoef(const KCSlot& s) {
  ICoef c;
  c.x0 = s.c0;
  c.x1 = s.c1;
  c.x2 = (uint64_t)((int64_t)s.c1 >> 63);
  return c;
}

// ---- K2: LSD radix sort (onesweep) ------------------------------------------
// One upfront histogram kernel gives every pass's global digit counts (the
// multiset of keys is the same for all passes).  Each pass is then a single
// kernel: tiles are claimed in launch order through a counter, rank their
// items stably with warp ballots (no shared-memory atomics), publish per-digit
// tile counts and find their exclusive prefix by decoupled look-back over the
// previous tiles, then scatter through shared memory so that global writes of
// equal digits are contiguous.
constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
#ifndef PGPU_RS_MINB
#define PGPU_RS_MINB 3
#endif
#ifndef PGPU_RS_IPT
#define PGPU_RS_IPT 12
#endif
#ifndef PGPU_RS_LOOKBACK
#define PGPU_RS_LOOKBACK 4
#endif
#ifndef PGPU_RS_BACKOFF
#define PGPU_RS_BACKOFF 1
#endif
constexpr int kRsIpt = PGPU_RS_IPT;                // items per thread per tile
constexpr int kRsTile = kRsThreads * kRsIpt;       // 4096
constexpr int kRsDigits = 256;
constexpr int kRsMaxPasses = 8;
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lanes holding the same 8-bit digit (restricted to `valid` lanes).
__device__ __forceinline__ unsigned digit_peers(unsigned d, unsigned valid) {
  unsigned peers = valid;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    unsigned bit = (d >> b) & 1u;
    unsigned bal = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? bal : ~bal;
  }
  return peers;
}

// ghist[p][d]: number of keys whose digit p is d, for all passes at once.
template <typename KT>
__global__ void __launch_bounds__(kRsThreads)
k_rs_hist_all(const KT* __restrict__ keys, uint64_t n, int npass, unsigned int* __restrict__ ghist) {
  __shared__ uint32_t h[kRsMaxPasses][kRsDigits];
  for (int k = threadIdx.x; k < kRsMaxPasses * kRsDigits; k += blockDim.x) (&h[0][0])[k] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint64_t idx = base + threadIdx.x;
    const bool ok = idx < n;
    const uint64_t k = ok ? (uint64_t)keys[idx] : 0ull;
    const unsigned valid = __ballot_sync(0xffffffffu, ok);
    for (int p = 0; p < npass; ++p) {
      const unsigned d = (unsigned)(k >> (8 * p)) & 0xffu;
      const unsigned peers = __match_any_sync(0xffffffffu, ok ? d : 0x100u) & valid;
      // one leader per digit group: shared-memory atomic add per group (few)
      if (ok && (peers & lanemask_lt()) == 0) atomicAdd(&h[p][d], (uint32_t)__popc(peers));
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < npass * kRsDigits; k += blockDim.x)
    if ((&h[0][0])[k]) atomicAdd(ghist + k, (&h[0][0])[k]);
}

// Exclusive scan of each pass's 256 counts, in place (one block).
__global__ void __launch_bounds__(kRsDigits) k_rs_hist_scan(unsigned int* ghist, int npass) {
  __shared__ uint32_t sh[33];
  for (int p = 0; p < npass; ++p) {
    uint32_t v = ghist[p * kRsDigits + threadIdx.x];
    uint32_t tot;
    uint32_t ex = block_excl_scan(v, sh, &tot);
    ghist[p * kRsDigits + threadIdx.x] = ex;
  }
}

#ifndef PGPU_RS_MINB32
#define PGPU_RS_MINB32 4
#endif
template <typename KT, typename VT = uint64_t>
__global__ void __launch_bounds__(kRsThreads, sizeof(VT) == 4 ? PGPU_RS_MINB32 : PGPU_RS_MINB)
k_rs_onesweep(const KT* __restrict__ kin, const VT* __restrict__ vin, KT* __restrict__ kout,
              VT* __restrict__ vout, uint64_t n, int shift, const unsigned int* __restrict__ gbase,
              unsigned long long* status, unsigned int* tile_ctr) {
  extern __shared__ __align__(16) uint8_t rs_smem[];
  VT* sval = reinterpret_cast<VT*>(rs_smem);                                   // [kRsTile]
  KT* skey = reinterpret_cast<KT*>(rs_smem + sizeof(VT) * kRsTile);            // [kRsTile]
  __shared__ uint32_t wcnt[kRsWarps][kRsDigits];
  __shared__ uint32_t tstart[kRsDigits];
  __shared__ uint32_t ttot[kRsDigits];
  __shared__ unsigned long long gpre[kRsDigits];
  __shared__ uint32_t shs[33];
  __shared__ uint32_t tile_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);
  for (int k = threadIdx.x; k < kRsWarps * kRsDigits; k += blockDim.x) (&wcnt[0][0])[k] = 0;
  __syncthreads();
  const uint32_t t = tile_s;
  const uint64_t t0 = (uint64_t)t * kRsTile;
  const uint64_t end = t0 + kRsTile < n ? t0 + kRsTile : n;
  KT key[kRsIpt];
  VT val[kRsIpt];
  uint32_t rank[kRsIpt];
  unsigned dig[kRsIpt];
  // warp w owns tile items [w*512, (w+1)*512): warp-major order is input order
#pragma unroll
  for (int k = 0; k < kRsIpt; ++k) {
    const uint64_t idx = t0 + (uint64_t)w * (32 * kRsIpt) + k * 32 + lane;
    const bool ok = idx < end;
    key[k] = ok ? kin[idx] : KT(0);
    val[k] = ok ? vin[idx] : VT(0);
  }
#pragma unroll
  for (int k = 0; k < kRsIpt; ++k) {
    const uint64_t idx = t0 + (uint64_t)w * (32 * kRsIpt) + k * 32 + lane;
    const bool ok = idx < end;
    dig[k] = ok ? (unsigned)((uint64_t)key[k] >> shift) & 0xffu : 0u;
    const unsigned peers = __match_any_sync(0xffffffffu, ok ? dig[k] : 0x100u);
    const uint32_t c = ok ? wcnt[w][dig[k]] : 0u;
    __syncwarp();
    rank[k] = c + __popc(peers & lt);
    if (ok && (peers & lt) == 0) wcnt[w][dig[k]] = c + __popc(peers);
    __syncwarp();
    if (!ok) dig[k] = 0xffffffffu;
  }
  __syncthreads();
  // per digit: exclusive over warps, tile total, then the decoupled look-back
  {
    const int d = threadIdx.x;  // kRsThreads == kRsDigits
    uint32_t sum = 0;
#pragma unroll
    for (int q = 0; q < kRsWarps; ++q) {
      const uint32_t c = wcnt[q][d];
      wcnt[q][d] = sum;
      sum += c;
    }
    ttot[d] = sum;
    volatile unsigned long long* st = status + (uint64_t)t * kRsDigits + d;
    if (t == 0) {
      *st = kFlagPre | sum;
      gpre[d] = 0;
    } else {
      *st = kFlagAgg | sum;
      unsigned long long excl = 0;
      int64_t k = (int64_t)t - 1;
#if PGPU_RS_LOOKBACK > 1
      // kLook predecessors per round trip: the chain of aggregate-only tiles
      // is walked kLook tiles at a time instead of one
      constexpr int kLook = PGPU_RS_LOOKBACK;
      unsigned backoff = 32;
      for (bool done = false; !done;) {
        unsigned long long v[kLook];
#pragma unroll
        for (int u = 0; u < kLook; ++u)
          v[u] = k - u >= 0 ? *(volatile unsigned long long*)(status + (uint64_t)(k - u) * kRsDigits + d)
                            : (2ull << 62);  // before tile 0: an inclusive zero
        bool progress = false;
#pragma unroll
        for (int u = 0; u < kLook; ++u) {
          if (done) break;
          const unsigned long long flag = v[u] & ~kValMask;
          if (flag == 0) break;  // not published yet: re-poll from here
          excl += v[u] & kValMask;
          --k;
          progress = true;
          if (flag == kFlagPre) done = true;
        }
        // a predecessor still ranking: back off instead of spinning, so the
        // issue slots go to the SM's other tiles
        if (!done && !progress && PGPU_RS_BACKOFF) {
          __nanosleep(backoff);
          backoff = backoff < 1024 ? backoff * 2 : 1024;
        }
      }
#else
      for (;;) {
        const unsigned long long v = *(volatile unsigned long long*)(status + (uint64_t)k * kRsDigits + d);
        const unsigned long long flag = v & ~kValMask;
        if (flag == 0) continue;  // predecessor not published yet
        excl += v & kValMask;
        if (flag == kFlagPre) break;
        --k;
      }
#endif
      *st = kFlagPre | (excl + sum);
      gpre[d] = excl;
    }
  }
  __syncthreads();
  {
    uint32_t v = ttot[threadIdx.x];
    uint32_t tot;
    uint32_t ex = block_excl_scan(v, shs, &tot);
    tstart[threadIdx.x] = ex;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kRsIpt; ++k) {
    if (dig[k] != 0xffffffffu) {
      const uint32_t pos = tstart[dig[k]] + wcnt[w][dig[k]] + rank[k];
      PGPU_ASSERT(pos < (uint32_t)kRsTile);
      skey[pos] = key[k];
      sval[pos] = val[k];
    }
  }
  __syncthreads();
  const uint32_t tn = (uint32_t)(end - t0);
  for (uint32_t q = threadIdx.x; q < tn; q += blockDim.x) {
    const KT kk = skey[q];
    const unsigned d = (unsigned)((uint64_t)kk >> shift) & 0xffu;
    const uint64_t g = (uint64_t)gbase[d] + gpre[d] + (q - tstart[d]);
    PGPU_ASSERT(g < n);
    kout[g] = kk;
    vout[g] = sval[q];
  }
}

// ---- K2 (super-tile passes): count / column scan / scatter -------------------
// The onesweep's decoupled look-back walks every predecessor tile still in
// flight (~600 on the GPU): on MP n=25 batches its spinning was ~90% of the
// pass's instructions and the pass ran at ~2 TB/s.  Here a pass is
//   RS1 k_rs_count    per super-tile (sup consecutive tiles) digit counts,
//                     digit-major cnt[d][st]; reads the keys only
//   RS2 k_rs_colscan  per digit: exclusive scan over the super-tiles (in
//                     place) and the digit total
//   RS3 k_rs_scatter  one CTA per super-tile: digit bases from the totals and
//                     its column prefix, then its tiles in order -- rank each
//                     tile stably (warp-major, __match_any_sync), stage it in
//                     shared memory by digit, write each digit's run at the
//                     running offset.  No inter-CTA waiting at all.
// Stable like the onesweep: tiles in order inside a super-tile, super-tiles in
// order through the column prefix, input order inside a tile.
#ifndef PGPU_RS_SUPER
#define PGPU_RS_SUPER 8
#endif
#ifndef PGPU_RS_MATCH
#define PGPU_RS_MATCH 1  // 1: __match_any_sync peers; 0: eight ballots
#endif
constexpr int kRsSuper = PGPU_RS_SUPER;
constexpr uint64_t kRsSuperItems = (uint64_t)kRsSuper * kRsTile;

template <typename KT>
__global__ void __launch_bounds__(kRsThreads)
k_rs_count(const KT* __restrict__ keys, uint64_t n, int shift, uint32_t nst, uint32_t sup,
           uint32_t* __restrict__ cnt) {
  // one histogram per warp, plain shared-memory atomics: after the first
  // pass the digits of a warp's 32 keys rarely collide, and a warp-level
  // match per key made the pass MIO-bound (match + atomic per key)
  __shared__ uint32_t h[kRsWarps][kRsDigits];
  const uint32_t st = blockIdx.x;
  const int w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < kRsWarps * kRsDigits; k += blockDim.x) (&h[0][0])[k] = 0;
  __syncthreads();
  const uint64_t b0 = (uint64_t)st * sup * kRsTile;
  const uint64_t b1 = b0 + (uint64_t)sup * kRsTile < n ? b0 + (uint64_t)sup * kRsTile : n;
  // 16-byte loads (V keys per thread per round; b0 is a multiple of V and the
  // arrays are 256-byte aligned)
  constexpr int V = 16 / sizeof(KT);
  using Vec = typename std::conditional<sizeof(KT) == 4, uint4, ulonglong2>::type;
  const Vec* kv = reinterpret_cast<const Vec*>(keys + b0);
  const uint64_t nv = (b1 - b0 + V - 1) / V;
  uint32_t* hw = h[w];
#pragma unroll 4
  for (uint64_t vi = threadIdx.x; vi < nv; vi += kRsThreads) {
    if (b0 + (vi + 1) * V <= b1) {
      const Vec x = kv[vi];
      if constexpr (sizeof(KT) == 4) {
        atomicAdd(&hw[(x.x >> shift) & 0xffu], 1u);
        atomicAdd(&hw[(x.y >> shift) & 0xffu], 1u);
        atomicAdd(&hw[(x.z >> shift) & 0xffu], 1u);
        atomicAdd(&hw[(x.w >> shift) & 0xffu], 1u);
      } else {
        atomicAdd(&hw[(unsigned)(x.x >> shift) & 0xffu], 1u);
        atomicAdd(&hw[(unsigned)(x.y >> shift) & 0xffu], 1u);
      }
    } else {
      for (int u = 0; u < V; ++u) {
        const uint64_t i = b0 + vi * V + u;
        if (i < b1) atomicAdd(&hw[(unsigned)((uint64_t)keys[i] >> shift) & 0xffu], 1u);
      }
    }
  }
  __syncthreads();
  uint32_t tot = 0;
#pragma unroll
  for (int q = 0; q < kRsWarps; ++q) tot += h[q][threadIdx.x];
  cnt[(uint64_t)threadIdx.x * nst + st] = tot;
}

// CTA d: exclusive scan of cnt[d][0, nst) in place; tot[d] = the digit's total
__global__ void __launch_bounds__(1024) k_rs_colscan(uint32_t* __restrict__ cnt, uint32_t nst,
                                                     uint32_t* __restrict__ tot) {
  __shared__ uint32_t sh[33];
  uint32_t* row = cnt + (uint64_t)blockIdx.x * nst;
  uint32_t carry = 0;
  constexpr int C = 4;
  for (uint32_t base = 0; base < nst; base += blockDim.x * C) {
    const uint32_t i0 = base + threadIdx.x * C;
    uint32_t v[C], sum = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      v[c] = i0 + c < nst ? row[i0 + c] : 0u;
      sum += v[c];
    }
    uint32_t t;
    uint32_t ex = block_excl_scan(sum, sh, &t) + carry;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (i0 + c < nst) row[i0 + c] = ex;
      ex += v[c];
    }
    carry += t;
  }
  if (threadIdx.x == 0) tot[blockIdx.x] = carry;
}

#ifndef PGPU_RS_SCAT_MINB
#define PGPU_RS_SCAT_MINB 3
#endif
template <typename KT, typename VT = uint64_t>
__global__ void __launch_bounds__(kRsThreads, PGPU_RS_SCAT_MINB)
k_rs_scatter(const KT* __restrict__ kin, const VT* __restrict__ vin, KT* __restrict__ kout,
             VT* __restrict__ vout, uint64_t n, int shift, uint32_t nst, uint32_t sup,
             const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ tot) {
  extern __shared__ __align__(16) uint8_t rs_smem[];
  VT* sval = reinterpret_cast<VT*>(rs_smem);                         // [kRsTile]
  KT* skey = reinterpret_cast<KT*>(rs_smem + sizeof(VT) * kRsTile);  // [kRsTile]
  __shared__ uint32_t wcnt[kRsWarps][kRsDigits];
  __shared__ uint32_t tstart[kRsDigits];
  __shared__ uint32_t ttot[kRsDigits];
  __shared__ unsigned long long run[kRsDigits];  // next output position of each digit
  __shared__ uint32_t shs[33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt();
  const uint32_t st = blockIdx.x;
  {  // digit bases: totals of the smaller digits + this super-tile's column prefix
    const uint32_t d = threadIdx.x;
    uint32_t t;
    const uint32_t ex = block_excl_scan(tot[d], shs, &t);
    run[d] = (unsigned long long)ex + cnt[(uint64_t)d * nst + st];
  }
  const uint64_t s0 = (uint64_t)st * sup * kRsTile;
  // The next tile is copied into a shared-memory buffer with cp.async while
  // this one is ranked and scattered (no registers held for it, so three
  // CTAs fit an SM).  16-byte chunks; a partial last tile is zero-filled.
  KT* pkey = reinterpret_cast<KT*>(rs_smem + (sizeof(KT) + sizeof(VT)) * kRsTile);  // [kRsTile]
  VT* pval = reinterpret_cast<VT*>(rs_smem + (2 * sizeof(KT) + sizeof(VT)) * kRsTile);
  auto prefetch = [&](uint64_t t0) {
    const uint64_t end = t0 + kRsTile < n ? t0 + kRsTile : n;
    constexpr int KC = 16 / sizeof(KT), VC = 16 / sizeof(VT);
    for (int c = threadIdx.x; c < kRsTile / KC; c += kRsThreads) {
      const uint64_t i = t0 + (uint64_t)c * KC;
      const int bytes = i >= end ? 0 : (int)(((uint64_t)KC < end - i ? (uint64_t)KC : end - i) * sizeof(KT));
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(pkey + c * KC);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(dst), "l"(kin + (bytes ? i : 0)), "r"(bytes));
    }
    for (int c = threadIdx.x; c < kRsTile / VC; c += kRsThreads) {
      const uint64_t i = t0 + (uint64_t)c * VC;
      const int bytes = i >= end ? 0 : (int)(((uint64_t)VC < end - i ? (uint64_t)VC : end - i) * sizeof(VT));
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(pval + c * VC);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(dst), "l"(vin + (bytes ? i : 0)), "r"(bytes));
    }
    asm volatile("cp.async.commit_group;");
  };
  if (s0 < n) prefetch(s0);
  KT key[kRsIpt];
  VT val[kRsIpt];
  for (uint32_t tl = 0; tl < sup; ++tl) {
    const uint64_t t0 = s0 + (uint64_t)tl * kRsTile;
    if (t0 >= n) break;
    const uint64_t end = t0 + kRsTile < n ? t0 + kRsTile : n;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // the tile is in the buffer for every thread
#pragma unroll
    for (int k = 0; k < kRsIpt; ++k) {
      const int q = w * (32 * kRsIpt) + k * 32 + lane;
      key[k] = pkey[q];
      val[k] = pval[q];
    }
    for (int k = threadIdx.x; k < kRsWarps * kRsDigits; k += blockDim.x) (&wcnt[0][0])[k] = 0;
    __syncthreads();  // buffer read by all: refill it with the next tile
    if (tl + 1 < sup && t0 + kRsTile < n) prefetch(t0 + kRsTile);
    uint32_t rank[kRsIpt];
    unsigned dig[kRsIpt];
#pragma unroll
    for (int k = 0; k < kRsIpt; ++k) {
      const uint64_t idx = t0 + (uint64_t)w * (32 * kRsIpt) + k * 32 + lane;
      const bool ok = idx < end;
      dig[k] = ok ? (unsigned)((uint64_t)key[k] >> shift) & 0xffu : 0u;
#if PGPU_RS_MATCH
      const unsigned peers = __match_any_sync(0xffffffffu, ok ? dig[k] : 0x100u);
#else
      const unsigned peers = digit_peers(dig[k], __ballot_sync(0xffffffffu, ok));  // (used for valid lanes only)
#endif
      const uint32_t c = ok ? wcnt[w][dig[k]] : 0u;
      __syncwarp();
      rank[k] = c + __popc(peers & lt);
      if (ok && (peers & lt) == 0) wcnt[w][dig[k]] = c + __popc(peers);
      __syncwarp();
      if (!ok) dig[k] = 0xffffffffu;
    }
    __syncthreads();
    {  // per digit: exclusive over warps and the tile total
      const int d = threadIdx.x;
      uint32_t sum = 0;
#pragma unroll
      for (int q = 0; q < kRsWarps; ++q) {
        const uint32_t c = wcnt[q][d];
        wcnt[q][d] = sum;
        sum += c;
      }
      ttot[d] = sum;
      uint32_t t;
      tstart[d] = block_excl_scan(sum, shs, &t);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRsIpt; ++k) {
      if (dig[k] != 0xffffffffu) {
        const uint32_t pos = tstart[dig[k]] + wcnt[w][dig[k]] + rank[k];
        PGPU_ASSERT(pos < (uint32_t)kRsTile);
        skey[pos] = key[k];
        sval[pos] = val[k];
      }
    }
    __syncthreads();
    const uint32_t tn = (uint32_t)(end - t0);
    for (uint32_t q = threadIdx.x; q < tn; q += blockDim.x) {
      const KT kk = skey[q];
      const unsigned d = (unsigned)((uint64_t)kk >> shift) & 0xffu;
      const uint64_t g = run[d] + (q - tstart[d]);
      PGPU_ASSERT(g < n);
      kout[g] = kk;
      vout[g] = sval[q];
    }
    __syncthreads();
    run[threadIdx.x] += ttot[threadIdx.x];
  }
}

// ---- K3: run-length heads -> segment starts ---------------------------------
// k_head_scan<KT, false> (scan.cuh): one pass over the sorted keys.

// ---- K4: segment reduce (one owner per output term) -------------------------
// G lanes own one segment (G = 1, 2, ..., 32, picked from the mean segment
// length): they stride over its pairs with coalesced record loads, then fold
// their exact partial sums with shuffles (limb adds modulo 2^(64 NL); the
// proven bound keeps the sum below 2^(64 NL - 1)).  Integer sums are
// order-independent, so any G gives the same result.
template <typename KT, int NL, int CK, int G>
__global__ void __launch_bounds__(256)
k_seg_reduce_int(const KT* __restrict__ keys, const uint64_t* __restrict__ vals,
                 const uint32_t* __restrict__ starts, uint32_t nseg, const void* __restrict__ ac,
                 const void* __restrict__ bc, uint64_t KL, KeyPlan P, uint64_t* __restrict__ oexp,
                 uint64_t* __restrict__ ocoef, uint32_t* __restrict__ onz) {
  const uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const uint32_t g = threadIdx.x % G;
  const bool live = s < nseg;  // whole groups are live or not; every lane reaches the shuffles
  const uint32_t p0 = live ? starts[s] : 0u, p1 = live ? starts[s + 1] : 0u;
  Limbs<NL> acc;
  limbs_zero(acc);
  for (uint32_t p = p0 + g; p < p1; p += G) {
    uint64_t v = vals[p];
    ICoef a = load_icoef<CK>(ac, (int64_t)(v >> 32));
    ICoef b = load_icoef<CK>(bc, (int64_t)(v & 0xffffffffu));
    limbs_add(acc, imul<NL, CK>(a, b));
  }
  if constexpr (G > 1) {
#pragma unroll
    for (int d = G / 2; d >= 1; d >>= 1) {
      Limbs<NL> o;
#pragma unroll
      for (int k = 0; k < NL; ++k) o.w[k] = __shfl_down_sync(0xffffffffu, acc.w[k], d, G);
      limbs_add(acc, o);
    }
  }
  if (!live || g != 0) return;
  oexp[s] = expand_key((uint64_t)keys[p0] + KL, P);
#pragma unroll
  for (int k = 0; k < NL; ++k) ocoef[(uint64_t)s * NL + k] = acc.w[k];
  onz[s] = limbs_nonzero(acc) ? 1u : 0u;
}

template <typename KT>
__global__ void __launch_bounds__(256)
k_seg_reduce_f64(const KT* __restrict__ keys, const uint64_t* __restrict__ vals,
                 const uint32_t* __restrict__ starts, uint32_t nseg, const double* __restrict__ ac,
                 const double* __restrict__ bc, uint64_t KL, KeyPlan P, uint64_t* __restrict__ oexp,
                 double* __restrict__ ocoef, uint32_t* __restrict__ onz) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  uint32_t p0 = starts[s], p1 = starts[s + 1];
  uint64_t v = vals[p0];
  // reference order: acc = a_i*b_j, then acc += a_i'*b_j' for increasing i'
  double acc = __dmul_rn(__ldg(ac + (v >> 32)), __ldg(bc + (v & 0xffffffffu)));
  for (uint32_t p = p0 + 1; p < p1; ++p) {
    v = vals[p];
    acc = __dadd_rn(acc, __dmul_rn(__ldg(ac + (v >> 32)), __ldg(bc + (v & 0xffffffffu))));
  }
  oexp[s] = expand_key((uint64_t)keys[p0] + KL, P);
  ocoef[s] = acc;
  onz[s] = (acc != 0.0) ? 1u : 0u;  // NaN != 0 -> kept, +-0 dropped (merge.py:63)
}

// K4 on j-records: the segment's key gives every pair's a-term through the
// key/coefficient hash (a_i = key + KL - b_j), then the same folds as above.
#ifndef PGPU_SEG_UNROLL
#define PGPU_SEG_UNROLL 1  // MP n=25 reduce 224 ms at 2, 238 at 4, 213 at 1; MP n=12 equal
#endif
template <typename RT, int NL, int CK, int G>
__global__ void __launch_bounds__(256)
k_seg_reduce_int_j(const RT* __restrict__ keys, const uint32_t* __restrict__ vals,
                   const uint32_t* __restrict__ starts, uint32_t nseg, const KCSlot* __restrict__ brec,
                   KCHash ahash, uint64_t KL, KeyPlan P, uint64_t* __restrict__ oexp,
                   uint64_t* __restrict__ ocoef, uint32_t* __restrict__ onz) {
  const uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const uint32_t g = threadIdx.x % G;
  const bool live = s < nseg;
  const uint32_t p0 = live ? starts[s] : 0u, p1 = live ? starts[s + 1] : 0u;
  const uint64_t key = live ? (uint64_t)keys[p0] + KL : 0ull;
  Limbs<NL> acc;
  limbs_zero(acc);
  uint32_t p = p0 + g;
  // PGPU_SEG_UNROLL pairs per iteration: every gather of each is issued before
  // any is used (three dependent loads per pair: column, b record, a slot)
  constexpr int U = PGPU_SEG_UNROLL;
  for (; p + (U - 1) * G < p1; p += U * G) {
    uint32_t j[U];
    KCSlot b[U], a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) j[u] = vals[p + u * G];
#pragma unroll
    for (int u = 0; u < U; ++u) b[u] = brec[j[u]];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = ahash.find(key - b[u].key);
#pragma unroll
    for (int u = 0; u < U; ++u) limbs_add(acc, imul<NL, CK>(kc_icoef<CK>(a[u]), kc_icoef<CK>(b[u])));
  }
  for (; p < p1; p += G) {
    const KCSlot b = brec[vals[p]];
    const KCSlot a = ahash.find(key - b.key);
    limbs_add(acc, imul<NL, CK>(kc_icoef<CK>(a), kc_icoef<CK>(b)));
  }
  if constexpr (G > 1) {
#pragma unroll
    for (int d = G / 2; d >= 1; d >>= 1) {
      Limbs<NL> o;
#pragma unroll
      for (int k = 0; k < NL; ++k) o.w[k] = __shfl_down_sync(0xffffffffu, acc.w[k], d, G);
      limbs_add(acc, o);
    }
  }
  if (!live || g != 0) return;
  oexp[s] = expand_key(key, P);
#pragma unroll
  for (int k = 0; k < NL; ++k) ocoef[(uint64_t)s * NL + k] = acc.w[k];
  onz[s] = limbs_nonzero(acc) ? 1u : 0u;
}

template <typename RT>
__global__ void __launch_bounds__(256)
k_seg_reduce_f64_j(const RT* __restrict__ keys, const uint32_t* __restrict__ vals,
                   const uint32_t* __restrict__ starts, uint32_t nseg, const KCSlot* __restrict__ brec,
                   KCHash ahash, uint64_t KL, KeyPlan P, uint64_t* __restrict__ oexp, double* __restrict__ ocoef,
                   uint32_t* __restrict__ onz) {
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const uint32_t p0 = starts[s], p1 = starts[s + 1];
  const uint64_t key = (uint64_t)keys[p0] + KL;
  // reference order: the stable sort kept generation order, i.e. increasing i
  double acc = 0.0;
  for (uint32_t p = p0; p < p1; ++p) {
    const KCSlot b = brec[vals[p]];
    const KCSlot a = ahash.find(key - b.key);
    const double pr = __dmul_rn(__longlong_as_double((long long)a.c0), __longlong_as_double((long long)b.c0));
    acc = p == p0 ? pr : __dadd_rn(acc, pr);
  }
  oexp[s] = expand_key(key, P);
  ocoef[s] = acc;
  onz[s] = (acc != 0.0) ? 1u : 0u;  // NaN != 0 -> kept, +-0 dropped (merge.py:63)
}

// ---- K5: zero-coefficient compaction ---------------------------------------
struct FlagGen {
  const uint32_t* f;
  __device__ uint32_t operator()(uint64_t i) const { return f[i]; }
};

struct CompactOut {
  const uint64_t* iexp;
  const uint64_t* icoef;   // limbs (f64 viewed as one u64 limb)
  int nl;
  uint64_t* oexp;
  uint64_t* ocoef;
  __device__ void operator()(uint64_t i, uint32_t ex, uint32_t v) const {
    if (!v) return;
    oexp[ex] = iexp[i];
    for (int k = 0; k < nl; ++k) ocoef[(uint64_t)ex * nl + k] = icoef[i * nl + k];
  }
};

}  // namespace pgpu
