// polymul_b200.cu -- C ABI and host orchestration of the B200 sparse
// polynomial multiplier (see include/polymul_b200.h).
//
// One call = one product, the reference `parmul.mul` (parmul.py:91-109):
//   1. operand checks: compatible/zero handled by the Python mirror;
//      exponent-field fit (check_product_fits, core.py:365-385) and the exact
//      coefficient width are proven here from device statistics;
//   2. compaction of packed exponents into short order-preserving keys;
//   3. the [lo, hi) packed range (split= lower bound, cluster range) becomes a
//      compact key range [KL, KH);
//   4. either the dense path (dense_path.cuh: sumset bytemap, per-interval
//      private accumulators) or the general sort path (sort_path.cuh);
//   5. zero-sum compaction and hand-back of (exps, coeffs) in ascending order
//      (concat, merge.py:164-173).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/polymul_b200.h"
#include "common.cuh"
#include "bucket_path.cuh"
#include "dense_path.cuh"
#include "format.cuh"
#include "prep.cuh"
#include "scan.cuh"
#include "small_path.cuh"
#include "sort_path.cuh"

using namespace pgpu;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

struct Status {
  int code = PGPU_OK;
};

#define CUDA_TRY(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      return fail(e_ == cudaErrorMemoryAllocation ? PGPU_ENOMEM : PGPU_ECUDA,          \
                  "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define TRY(x)                 \
  do {                         \
    int r_ = (x);              \
    if (r_ != PGPU_OK) return r_; \
  } while (0)

#define LAUNCHED(k) (ctx.launches += (k))

// Per-device state: library stream, a retained stream-ordered pool, and a
// persistent scratch workspace (bump-allocated per call, grown between calls).
struct DeviceState {
  bool init = false;
  cudaStream_t stream = nullptr;
  uint8_t* ws = nullptr;
  size_t ws_cap = 0;
  size_t ws_want = 0;  // high-water mark requested by previous calls
  size_t mem_free0 = 0, mem_total = 0;  // device memory at first use (cudaMemGetInfo is
                                        // slow and occasionally blocks for milliseconds)
  std::mutex mu;       // one product per device at a time uses the workspace
  uint8_t* stage = nullptr;  // pinned staging for small host operands (copy_in_small)
  uint8_t* rb = nullptr;     // pinned readback of small device values (counts, statistics)
};
constexpr size_t kReadback = 64 << 10;
std::mutex g_mu;
DeviceState g_dev[64];

int device_setup(int dev, cudaStream_t* st) {
  CUDA_TRY(cudaSetDevice(dev));
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceState& d = g_dev[dev & 63];
  if (!d.init) {
    CUDA_TRY(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = ~0ull;
    CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    CUDA_TRY(cudaMemGetInfo(&d.mem_free0, &d.mem_total));
    CUDA_TRY(cudaMallocHost((void**)&d.rb, kReadback));
    d.init = true;
  }
  *st = d.stream;
  return PGPU_OK;
}

// Kernel attributes are per device context: the opt-in shared-memory size is
// set once per (kernel, device), and occupancy queries are cached per kernel.
std::mutex g_attr_mu;
std::set<std::pair<const void*, int>> g_attr_done;
std::map<std::pair<const void*, size_t>, int> g_occ;

template <typename K>
void smem_attr(K kern, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (g_attr_done.insert({(const void*)kern, dev}).second)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// resident CTAs per SM (>= 1)
template <typename K>
int occupancy(K kern, int threads, size_t smem) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto it = g_occ.find({(const void*)kern, smem});
  if (it != g_occ.end()) return it->second;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 1;
  }
  per_sm = std::max(per_sm, 1);
  g_occ[{(const void*)kern, smem}] = per_sm;
  return per_sm;
}

// The ABI never leaves the caller's thread on another device (torch keeps its
// own notion of the current device).
struct DeviceRestore {
  int prev = -1;
  DeviceRestore() {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
  }
  ~DeviceRestore() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

constexpr size_t kWorkspaceMaxItem = 1ull << 30;  // larger buffers bypass the workspace
constexpr size_t kWorkspaceMax = 16ull << 30;     // workspace never grows beyond this

// Scratch allocator.  Requests are bump-allocated from the device workspace;
// when it is too small the request falls back to cudaMallocAsync and the
// workspace is regrown after the call.  Memory handed to the caller always
// comes from cudaMallocAsync (it outlives the call).
struct Arena {
  cudaStream_t st;
  DeviceState* dev = nullptr;
  size_t used = 0;
  size_t requested = 0;
  std::vector<void*> ptrs;  // cudaMallocAsync allocations owned by the arena
  uint8_t* blk = nullptr;   // caller-provided block (batch scratch): any item size
  size_t blk_cap = 0;
  explicit Arena(cudaStream_t s, DeviceState* d = nullptr, size_t base = 0)
      : st(s), dev(d), used(base), requested(base) {}
  Arena(cudaStream_t s, uint8_t* block, size_t cap) : st(s), blk(block), blk_cap(cap) {}
  ~Arena() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    if (dev && requested > dev->ws_want) dev->ws_want = requested;
  }
  template <typename T>
  int alloc(T** p, size_t count) {
    size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    bytes = (bytes + 255) & ~size_t(255);
    if (blk) {
      if (used + bytes <= blk_cap) {
        *p = reinterpret_cast<T*>(blk + used);
        used += bytes;
        return PGPU_OK;
      }
      return alloc_fresh(p, bytes);
    }
    if (bytes > kWorkspaceMaxItem) return alloc_fresh(p, bytes);  // big batch buffers: pool only
    requested += bytes;
    if (dev && dev->ws && used + bytes <= dev->ws_cap) {
      *p = reinterpret_cast<T*>(dev->ws + used);
      used += bytes;
      return PGPU_OK;
    }
    return alloc_fresh(p, bytes);
  }
  template <typename T>
  int alloc_out(T** p, size_t count) {  // caller-owned result buffer
    size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    return alloc_fresh(p, bytes);
  }
  template <typename T>
  int alloc_fresh(T** p, size_t bytes) {
    cudaError_t e = cudaMallocAsync((void**)p, bytes, st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(PGPU_ENOMEM, "device allocation of %zu bytes failed: %s", bytes,
                  cudaGetErrorString(e));
    }
    ptrs.push_back((void*)*p);
    return PGPU_OK;
  }
  bool owns(void* p) const { return std::find(ptrs.begin(), ptrs.end(), p) != ptrs.end(); }
  void release(void* p) {  // ownership moves to the caller
    ptrs.erase(std::remove(ptrs.begin(), ptrs.end(), p), ptrs.end());
  }
};

// Grow the workspace to the last call's high-water mark (between calls only).
int grow_workspace(DeviceState& d, cudaStream_t st) {
  if (d.ws_want <= d.ws_cap) return PGPU_OK;
  size_t freeb = 0, totb = 0;
  CUDA_TRY(cudaStreamSynchronize(st));
  if (d.ws) CUDA_TRY(cudaFree(d.ws));
  d.ws = nullptr;
  d.ws_cap = 0;
  CUDA_TRY(cudaMemGetInfo(&freeb, &totb));
  size_t want = std::min(d.ws_want + d.ws_want / 4, kWorkspaceMax);
  if (getenv("PGPU_DEBUG"))
    fprintf(stderr, "[pgpu] workspace grow %zu -> %zu bytes\n", d.ws_cap, want);
  if (want > freeb / 2) want = d.ws_want <= freeb / 2 ? d.ws_want : 0;  // keep room for the pool
  if (want == 0) return PGPU_OK;
  if (cudaMalloc((void**)&d.ws, want) != cudaSuccess) {
    cudaGetLastError();
    d.ws = nullptr;
    return PGPU_OK;  // fall back to per-call allocations
  }
  d.ws_cap = want;
  return PGPU_OK;
}

// Pinned host buffers for host-side results: D2H into page-locked memory runs
// at full PCIe/C2C speed, and reusing blocks avoids cudaMallocHost per call.
// Blocks are tagged in pgpu_result._owner and come back via pgpu_free_result.
struct PinnedPool {
  std::mutex mu;
  std::vector<std::pair<void*, size_t>> free_blocks;
  static constexpr size_t kMaxCached = 8;
  void* get(size_t bytes) {
    {
      std::lock_guard<std::mutex> lk(mu);
      size_t best = SIZE_MAX;
      int bi = -1;
      for (size_t k = 0; k < free_blocks.size(); ++k)
        if (free_blocks[k].second >= bytes && free_blocks[k].second < best) {
          best = free_blocks[k].second;
          bi = (int)k;
        }
      if (bi >= 0) {
        void* p = free_blocks[bi].first;
        free_blocks.erase(free_blocks.begin() + bi);
        return p;
      }
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    std::lock_guard<std::mutex> lk(mu);  // put() may run concurrently (no device lock there)
    sizes_[p] = bytes;
    return p;
  }
  void put(void* p) {
    std::lock_guard<std::mutex> lk(mu);
    if (free_blocks.size() >= kMaxCached) {
      cudaFreeHost(free_blocks.front().first);
      sizes_.erase(free_blocks.front().first);
      free_blocks.erase(free_blocks.begin());
    }
    free_blocks.push_back({p, sizes_[p]});
  }
  std::map<void*, size_t> sizes_;
};
PinnedPool g_pinned;
constexpr uintptr_t kPinnedTag = 0x50494e4e;  // result buffers come from g_pinned
constexpr uintptr_t kDevTag = 0x44455600;     // device result: kDevTag | device ordinal

// stream-ordered free of a device result on its own device's library stream
void free_device_ptr(void* p, void* owner) {
  if (!p) return;
  const uintptr_t tag = (uintptr_t)owner;
  if ((tag & ~uintptr_t(0xff)) == kDevTag) {
    const int dev = (int)(tag & 0xff);
    DeviceRestore dr;
    if (cudaSetDevice(dev) == cudaSuccess && g_dev[dev & 63].init) {
      cudaFreeAsync(p, g_dev[dev & 63].stream);
      return;
    }
    cudaGetLastError();
  }
  cudaFreeAsync(p, 0);
}

// Host timeline of one call (PGPU_TRACE=1): where the wall time of a product
// goes between launches and synchronisations.
struct Trace {
  bool on = false;
  int n = 0;
  const char* what[32];
  double t[32];
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
  }
  void at(const char* w) {
    if (on && n < 32) {
      what[n] = w;
      t[n++] = now();
    }
  }
  void dump() {
    if (!on || n < 2) return;
    fprintf(stderr, "[pgpu trace]");
    for (int k = 1; k < n; ++k) fprintf(stderr, " %s=%.3f", what[k], t[k] - t[k - 1]);
    fprintf(stderr, " total=%.3f ms\n", t[n - 1] - t[0]);
  }
};
thread_local Trace g_trace;

struct Timer {
  bool on = false;
  cudaStream_t st;
  int n = 0;
  cudaEvent_t ev[PGPU_NPHASE + 1];
  const char* names[PGPU_NPHASE] = {nullptr};
  float acc[PGPU_NPHASE] = {0};
  void start(cudaStream_t s, bool enable) {
    on = enable;
    st = s;
    if (!on) return;
    for (int k = 0; k <= PGPU_NPHASE; ++k) cudaEventCreate(&ev[k]);
    cudaEventRecord(ev[0], st);
  }
  // close phase k (phases may repeat across batches: times accumulate)
  void mark(int k, const char* name) {
    if (!on) return;
    names[k] = name;
    if (k + 1 > n) n = k + 1;
    cudaEventRecord(ev[PGPU_NPHASE], st);
    cudaEventSynchronize(ev[PGPU_NPHASE]);
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[0], ev[PGPU_NPHASE]);
    acc[k] += ms;
    std::swap(ev[0], ev[PGPU_NPHASE]);
  }
  void finish(pgpu_result* r) {
    if (!on) return;
    r->n_phase = n;
    for (int k = 0; k < n; ++k) {
      r->phase_ms[k] = acc[k];
      r->phase_name[k] = names[k];
    }
    for (int k = 0; k <= PGPU_NPHASE; ++k) cudaEventDestroy(ev[k]);
  }
};

struct Ctx {
  cudaStream_t st;
  Arena* ar;
  void* rh_key = nullptr;     // key/coefficient hash of operand a (sort path j-records: KCSlot[]), or null
  uint32_t rh_mask = 0;
  void* brec = nullptr;       // operand b as KCSlot[] (j-records)
  uint8_t* batch_blk = nullptr;  // one block reused by every batch of a product
  size_t batch_cap = 0;
  size_t mem_budget = 0;  // bytes this call may plan to use for large scratch
  Timer tm;
  int64_t launches = 0;
  int sms = 148;
  int device = 0;
  uint8_t* rb = nullptr;  // pinned readback area of the device (the device lock is held)
  size_t rb_used = 0;
  // pinned host slots for small device-to-host reads (a pageable destination
  // makes cudaMemcpyAsync a staged, synchronous copy: ~50 us each)
  template <typename T>
  T* pin(size_t n) {
    const size_t bytes = (n * sizeof(T) + 15) & ~size_t(15);
    if (!rb || rb_used + bytes > kReadback) return nullptr;
    T* p = reinterpret_cast<T*>(rb + rb_used);
    rb_used += bytes;
    return p;
  }
};

inline int grid_for(int64_t n, int threads, int cap) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

inline int bitlen64(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

// Everything the product needs once operands are on the device.
struct Problem {
  const uint64_t* aexp;
  const uint64_t* bexp;
  const void* acoef;
  const void* bcoef;
  uint32_t na, nb;
  int ck;          // coefficient kind
  int nl;          // integer result limbs (0 for f64)
  int need_bits;   // proven bound on |coefficient| bits + sign
  bool nonneg;     // no negative operand coefficient (unsigned products)
  KeyPlan P;
  bool k32;        // keys fit 32 bits
  void* ak;        // compact keys (uint32_t* or uint64_t*)
  void* bk;
  uint64_t KL, KH; // compact key range
  uint64_t kmin, kmax;  // smallest / largest compact key of any pair
};

// A finished slice of the result (device buffers owned by the arena).
struct Slice {
  uint64_t* exps;
  uint64_t* coef;  // limbs (f64 bit patterns when nl == 1 and ck == f64)
  uint64_t n;
};

// ---------------------------------------------------------------------------
// Row edges + exclusive offsets of a key range; returns the pair count.
// ---------------------------------------------------------------------------
template <typename KT>
int range_rows(Ctx& ctx, const Problem& pb, uint64_t KL, uint64_t KH, uint32_t** rlo,
               uint32_t** rhi, uint64_t** off, uint64_t* pairs) {
  TRY(ctx.ar->alloc(rlo, pb.na));
  TRY(ctx.ar->alloc(rhi, pb.na));
  k_edges<KT><<<grid_for(pb.na, 256, 1 << 30), 256, 0, ctx.st>>>(
      (const KT*)pb.ak, pb.na, (const KT*)pb.bk, pb.nb, KL, KH, *rlo, *rhi);
  LAUNCHED(1);
  if (!off) return PGPU_OK;  // the dense path needs the row windows only
  TRY(ctx.ar->alloc(off, pb.na));
  uint64_t* part;
  TRY(ctx.ar->alloc(&part, kMaxScanBlocks + 1));
  int g;
  LAUNCHED(device_scan<uint64_t>(pb.na, LenGen{*rlo, *rhi}, OffOut{*off}, part, &g, ctx.st));
  if (pairs) {
    uint64_t* p = ctx.pin<uint64_t>(1);
    CUDA_TRY(cudaMemcpyAsync(p ? p : pairs, part + g, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.st));
    CUDA_TRY(cudaStreamSynchronize(ctx.st));
    if (p) *pairs = *p;
  }
  return PGPU_OK;
}

template <typename KT>
int count_at(Ctx& ctx, const Problem& pb, const std::vector<uint64_t>& bounds,
             std::vector<uint64_t>& cum) {
  cum.assign(bounds.size(), 0);
  if (bounds.empty()) return PGPU_OK;
  uint64_t* db;
  unsigned long long* dc;
  TRY(ctx.ar->alloc(&db, bounds.size()));
  TRY(ctx.ar->alloc(&dc, bounds.size()));
  CUDA_TRY(cudaMemcpyAsync(db, bounds.data(), bounds.size() * 8, cudaMemcpyHostToDevice, ctx.st));
  CUDA_TRY(cudaMemsetAsync(dc, 0, bounds.size() * 8, ctx.st));
  for (size_t b0 = 0; b0 < bounds.size(); b0 += 65535) {
    unsigned nbnd = (unsigned)std::min<size_t>(65535, bounds.size() - b0);
    dim3 grid(grid_for(pb.na, 256, 64), nbnd);
    k_count_multi<KT><<<grid, 256, 0, ctx.st>>>((const KT*)pb.ak, pb.na, (const KT*)pb.bk, pb.nb,
                                                db + b0, dc + b0);
    LAUNCHED(1);
  }
  uint64_t* p = ctx.pin<uint64_t>(bounds.size());
  CUDA_TRY(cudaMemcpyAsync(p ? p : cum.data(), dc, bounds.size() * 8, cudaMemcpyDeviceToHost, ctx.st));
  CUDA_TRY(cudaStreamSynchronize(ctx.st));
  if (p) std::copy(p, p + bounds.size(), cum.begin());
  return PGPU_OK;
}

// Sort path driver (kernels in sort_path.cuh)
#include "sort_driver.inc"

// Bucket path driver (kernels in bucket_path.cuh)
#include "bucket_driver.inc"

// Memory this process can still use on device `dev`: free device memory plus
// what the stream-ordered pool holds reserved but unused (it retains freed
// blocks).  Queried only for large products: cudaMemGetInfo can stall.
size_t fresh_budget(int dev) {
  size_t f = 0, t = 0;
  if (cudaMemGetInfo(&f, &t) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaMemPool_t pool;
  uint64_t res = 0, used = 0;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  } else {
    cudaGetLastError();
  }
  return f + (res > used ? (size_t)(res - used) : 0);
}

template <typename KT>
int run_sort_path(Ctx& ctx, const Problem& pb, uint64_t total, std::vector<Slice>& slices,
                  bool try_bucket, int* nbucket, double cap_scale = 1.0) {
  // per pair: records x2 (key + i<<32|j), segment starts; the segment outputs
  // (<= pairs, usually far fewer) and scan scratch fit in the remaining slack
  uint64_t bpp = 2 * (sizeof(KT) + 8) + 4 + 8;
  size_t freeb = ctx.mem_budget;
  if (cap_scale < 1.0) {  // a retry after ENOMEM: the budget cached at first use was stale
    const size_t now = fresh_budget(ctx.device);
    if (now) freeb = std::min(freeb, now);
  }
  uint64_t cap = (uint64_t)(freeb * 0.55 * cap_scale) / bpp;
  if (cap > (1ull << 31)) cap = 1ull << 31;  // 32-bit positions inside a batch
  const char* env = getenv("PGPU_BATCH_CAP");
  if (env) cap = std::min<uint64_t>(cap, strtoull(env, nullptr, 10));
  std::vector<std::pair<uint64_t, uint64_t>> ranges;
  std::vector<uint64_t> counts;
  // wide operand keys: batches narrow enough for 32-bit record keys, unless
  // that would take more than a few dozen extra batches
  uint64_t max_span = 0;
  if (!pb.k32) {
    const uint64_t span = (pb.KH == ~0ull ? pb.kmax + 1 : pb.KH) - pb.KL;
    if ((span >> 32) <= 48 && !getenv("PGPU_NO_SPAN32")) max_span = 0xffffffffull;
  }
  TRY(plan_batches<KT>(ctx, pb, pb.KL, pb.KH, total, cap, ranges, counts, max_span));
  // Large products: 8-byte sort records (key, column j); the row of a pair is
  // recovered from its key through a hash of operand a's keys, built once here.
  // (Keys of a are distinct; the all-ones key marks empty slots, so it must be
  // out of range.)
  ctx.rh_key = nullptr;
  const uint64_t jrec_min = getenv("PGPU_JREC_MIN") ? strtoull(getenv("PGPU_JREC_MIN"), nullptr, 10)
                                                   : (1ull << 20);
  if (total >= jrec_min && pb.P.kbits < 64 && !getenv("PGPU_NO_JREC")) {
    // key/coefficient slots: a hash of operand a (load factor <= 1/4: ~1.2
    // probes per lookup; 18 MB for MP n=25, L2-resident), operand b in order
    uint32_t cap = 1;
    while (cap < 4 * pb.na) cap <<= 1;
    KCSlot *slots, *brec;
    TRY(ctx.ar->alloc(&slots, cap));
    TRY(ctx.ar->alloc(&brec, pb.nb));
    CUDA_TRY(cudaMemsetAsync(slots, 0xff, sizeof(KCSlot) * cap, ctx.st));
    const int ga = grid_for(pb.na, 256, 1 << 30), gb = grid_for(pb.nb, 256, 1 << 30);
    if (pb.ck == PGPU_I128) {
      k_kc_hash_build<KT, 2><<<ga, 256, 0, ctx.st>>>((const KT*)pb.ak, pb.acoef, pb.na, slots, cap - 1);
      k_kc_fill<KT, 2><<<gb, 256, 0, ctx.st>>>((const KT*)pb.bk, pb.bcoef, pb.nb, brec);
    } else {  // f64 bits and int64 share the one-word layout
      k_kc_hash_build<KT, 1><<<ga, 256, 0, ctx.st>>>((const KT*)pb.ak, pb.acoef, pb.na, slots, cap - 1);
      k_kc_fill<KT, 1><<<gb, 256, 0, ctx.st>>>((const KT*)pb.bk, pb.bcoef, pb.nb, brec);
    }
    LAUNCHED(2);
    ctx.rh_key = slots;
    ctx.rh_mask = cap - 1;
    ctx.brec = brec;
  }
  struct RowHashOff {
    Ctx& c;
    ~RowHashOff() { c.rh_key = nullptr; }
  } rh_off{ctx};
  // Products with several large batches: one scratch block sized for the
  // largest batch serves them all (per-batch pool allocations of tens of GB
  // made run times vary by up to 2x through physical remapping).
  uint64_t maxc = 0;
  for (uint64_t c : counts) maxc = std::max(maxc, c);
  const size_t blk_bytes = (size_t)maxc * bpp + (256ull << 20);
  if (ranges.size() > 1 && blk_bytes > (1ull << 30)) {
    if (cudaMallocAsync((void**)&ctx.batch_blk, blk_bytes, ctx.st) == cudaSuccess) {
      ctx.batch_cap = blk_bytes;
    } else {
      cudaGetLastError();
      ctx.batch_blk = nullptr;
    }
  }
  struct BlkFree {
    Ctx& c;
    ~BlkFree() {
      if (c.batch_blk) cudaFreeAsync(c.batch_blk, c.st);
      c.batch_blk = nullptr;
    }
  } blk_free{ctx};
  for (size_t r = 0; r < ranges.size(); ++r) {
    Slice s;
    bool done = false;
    if (try_bucket)
      TRY(bucket_range<KT>(ctx, pb, ranges[r].first, ranges[r].second, counts[r], &s, &done, ranges.size() == 1));
    if (done) ++*nbucket;
    else TRY(sort_range<KT>(ctx, pb, ranges[r].first, ranges[r].second, counts[r], &s));
    if (s.n) slices.push_back(s);
  }
  return PGPU_OK;
}

// Dense path driver (kernels in dense_path.cuh)
#include "dense_driver.inc"

// ---------------------------------------------------------------------------
int build_problem(Ctx& ctx, const pgpu_layout* lay, const pgpu_options* opt, Problem& pb,
                  const pgpu_options& o) {
  // layout -> KeyPlan (packed part)
  KeyPlan& P = pb.P;
  memset(&P, 0, sizeof P);
  P.nf = lay->nfields;
  P.order = lay->order;
  for (int f = 0; f < P.nf; ++f) {
    P.shift[f] = lay->shift[f];
    P.mask[f] = lay->width[f] >= 64 ? ~0ull : ((1ull << lay->width[f]) - 1);
  }
  OperandStats* dst;
  TRY(ctx.ar->alloc(&dst, 1));
  CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(OperandStats), ctx.st));
  int ga = grid_for(pb.na, 256, ctx.sms * 4), gb = grid_for(pb.nb, 256, ctx.sms * 4);
  double* dsum;
  TRY(ctx.ar->alloc(&dsum, ga + gb));
  if (o.coef_kind == PGPU_F64) {
    k_stats<0><<<ga, 256, 0, ctx.st>>>(pb.aexp, pb.acoef, pb.na, P, dst, 0, dsum);
    k_stats<0><<<gb, 256, 0, ctx.st>>>(pb.bexp, pb.bcoef, pb.nb, P, dst, 1, dsum + ga);
  } else if (o.coef_kind == PGPU_I64) {
    k_stats<1><<<ga, 256, 0, ctx.st>>>(pb.aexp, pb.acoef, pb.na, P, dst, 0, dsum);
    k_stats<1><<<gb, 256, 0, ctx.st>>>(pb.bexp, pb.bcoef, pb.nb, P, dst, 1, dsum + ga);
  } else {
    k_stats<2><<<ga, 256, 0, ctx.st>>>(pb.aexp, pb.acoef, pb.na, P, dst, 0, dsum);
    k_stats<2><<<gb, 256, 0, ctx.st>>>(pb.bexp, pb.bcoef, pb.nb, P, dst, 1, dsum + ga);
  }
  LAUNCHED(2);
  // range thresholds (packed) and operand ends ride the same round trip
  const uint64_t npairs = (uint64_t)pb.na * pb.nb;
  const bool small_only = o.lo == 0 && o.hi == ~0ull && npairs <= (uint64_t)kSmallPairs &&
                          !getenv("PGPU_NO_SMALL") && (o.path == PGPU_PATH_AUTO || o.path == PGPU_PATH_SMALL);
  uint64_t S[2] = {o.lo, o.hi};
  const bool need_thr[2] = {o.lo != 0, o.hi != ~0ull};
  unsigned long long* dthr;  // [0,1] thresholds, [2..5] operand ends
  TRY(ctx.ar->alloc(&dthr, 6));
  if (!small_only) {
    CUDA_TRY(cudaMemsetAsync(dthr, 0xff, 16, ctx.st));  // ~0: no pair reaches the bound
    for (int sdx = 0; sdx < 2; ++sdx) {
      if (!need_thr[sdx]) continue;
      k_threshold<<<grid_for(pb.na, 256, 1 << 30), 256, 0, ctx.st>>>(pb.aexp, pb.na, pb.bexp, pb.nb, S[sdx],
                                                                      dthr + sdx);
      LAUNCHED(1);
    }
    k_exp_ends<<<1, 32, 0, ctx.st>>>(pb.aexp, pb.na, pb.bexp, pb.nb, dthr + 2);
    LAUNCHED(1);
  }
  g_trace.at("stats_kernels");
  OperandStats hs;
  std::vector<double> hsum(ga + gb);
  OperandStats* hs_p = ctx.pin<OperandStats>(1);
  double* hsum_p = ctx.pin<double>(ga + gb);
  if (!hs_p || !hsum_p) {
    hs_p = &hs;
    hsum_p = hsum.data();
  }
  CUDA_TRY(cudaMemcpyAsync(hs_p, dst, sizeof hs, cudaMemcpyDeviceToHost, ctx.st));
  CUDA_TRY(cudaMemcpyAsync(hsum_p, dsum, 8ull * (ga + gb), cudaMemcpyDeviceToHost, ctx.st));
  unsigned long long thr_local[6];
  unsigned long long* thr = ctx.pin<unsigned long long>(6);
  if (!thr) thr = thr_local;
  if (!small_only) CUDA_TRY(cudaMemcpyAsync(thr, dthr, 48, cudaMemcpyDeviceToHost, ctx.st));
  g_trace.at("stats_launch");
  CUDA_TRY(cudaStreamSynchronize(ctx.st));
  g_trace.at("stats_sync");
  if (hs_p != &hs) {
    hs = *hs_p;
    std::copy(hsum_p, hsum_p + ga + gb, hsum.begin());
  }
  // rigorous upper bounds of sum|a_i| and sum|b_j|: device partials are rounded
  // up; the host sum gets the recursive-summation error margin on top
  double sa = 0, sb = 0;
  for (int k = 0; k < ga; ++k) sa += hsum[k];
  for (int k = 0; k < gb; ++k) sb += hsum[ga + k];
  sa *= 1.0 + 4.0 * (ga + gb + 2) * 1.1102230246251565e-16;
  sb *= 1.0 + 4.0 * (ga + gb + 2) * 1.1102230246251565e-16;
  pb.nonneg = !(hs.negative[0] || hs.negative[1]);
  if (hs.unsorted[0] || hs.unsorted[1])
    return fail(PGPU_EINVAL, "operand exponents are not strictly ascending packed words");
  // exponent fit (core.py:365-385): field sums must stay within the caps
  for (int f = 0; f < P.nf; ++f) {
    uint64_t cap = P.mask[f];
    if (f == 0) cap -= 1;  // grlex degree ceiling / lex top-field ceiling reserved
    uint64_t s = hs.fmax[0][f] + hs.fmax[1][f];
    if (s > cap || s < hs.fmax[0][f]) {
      return fail(PGPU_EEXPONENT, "product %s field %d can reach %llu, field range is 0..%llu",
                  (P.order == 0 && f == 0) ? "total degree" : "exponent", f,
                  (unsigned long long)s, (unsigned long long)cap);
    }
  }
  // exact coefficient width.  |c_k| <= sum over its pairs |a_i||b_j|, which is
  // <= min(na,nb)*max|a|*max|b| and <= min(sum|a|*max|b|, max|a|*sum|b|).
  pb.nl = 0;
  if (o.coef_kind != PGPU_F64) {
    int need = (int)hs.cbits[0] + (int)hs.cbits[1] + bitlen64(std::min(pb.na, pb.nb)) + 1;
    double ma, mb;
    memcpy(&ma, &hs.maxmag[0], 8);
    memcpy(&mb, &hs.maxmag[1], 8);
    const double rel = 1.0 + 4.0 * 1.1102230246251565e-16;  // the products below round once
    double bound = std::min(sa * mb, ma * sb) * rel;
    if (bound > 0 && std::isfinite(bound)) {
      int ex;
      frexp(bound, &ex);  // bound < 2^ex
      need = std::min(need, ex + 1);
    }
    pb.need_bits = need;
    if (getenv("PGPU_DEBUG"))
      fprintf(stderr, "[pgpu] coefficient bound: cbits %u+%u, sum|a| %.6g sum|b| %.6g max|a| %.6g max|b| %.6g -> %d bits\n",
              hs.cbits[0], hs.cbits[1], sa, sb, ma, mb, need);
    int nl = (need + 63) / 64;
    if (nl < 1) nl = 1;
    if (nl > 3)
      return fail(PGPU_ECOEFF, "exact coefficients may need %d bits; the widest accumulator is 192",
                  need);
    if (o.acc_limbs) {
      if (o.acc_limbs < nl)
        return fail(PGPU_ECOEFF, "requested %d-limb accumulator but the bound needs %d bits",
                    o.acc_limbs, need);
      nl = std::min(o.acc_limbs, 3);
    }
    pb.nl = nl;
  }
  // key compaction plan
  int pos = 0;
  P.dropped = (P.order == 0) ? P.nf - 1 : -1;
  for (int f = P.nf - 1; f >= 0; --f) {
    uint64_t s = hs.fmax[0][f] + hs.fmax[1][f];
    int cw = bitlen64(s);
    P.keep[f] = (cw > 0 && f != P.dropped) ? 1 : 0;
    P.cpos[f] = pos;
    P.cmask[f] = cw >= 64 ? ~0ull : ((1ull << cw) - 1);
    if (P.keep[f]) pos += cw;
  }
  P.kbits = pos;
  pb.k32 = pos <= 32;
  size_t ksz = pb.k32 ? 4 : 8;
  TRY(ctx.ar->alloc((uint8_t**)&pb.ak, ksz * pb.na));
  TRY(ctx.ar->alloc((uint8_t**)&pb.bk, ksz * (pb.nb + 128)));  // padded for unrolled loads
  if (pb.k32) {
    k_compact<uint32_t><<<ga, 256, 0, ctx.st>>>(pb.aexp, pb.na, P, (uint32_t*)pb.ak);
    k_compact<uint32_t><<<gb, 256, 0, ctx.st>>>(pb.bexp, pb.nb, P, (uint32_t*)pb.bk);
  } else {
    k_compact<uint64_t><<<ga, 256, 0, ctx.st>>>(pb.aexp, pb.na, P, (uint64_t*)pb.ak);
    k_compact<uint64_t><<<gb, 256, 0, ctx.st>>>(pb.bexp, pb.nb, P, (uint64_t*)pb.bk);
  }
  LAUNCHED(2);
  // packed [lo, hi) -> compact [KL, KH)
  pb.KL = 0;
  pb.KH = ~0ull;
  if (small_only && P.kbits + std::max(1, bitlen64(npairs - 1)) <= 63) {
    // the one-CTA path needs neither thresholds nor key ends
    pb.kmin = 0;
    pb.kmax = ~0ull;
    return PGPU_OK;
  }
  if (small_only) {  // key too wide for the one-CTA sort word: thresholds after all
    CUDA_TRY(cudaMemsetAsync(dthr, 0xff, 16, ctx.st));
    k_exp_ends<<<1, 32, 0, ctx.st>>>(pb.aexp, pb.na, pb.bexp, pb.nb, dthr + 2);
    LAUNCHED(1);
    CUDA_TRY(cudaMemcpyAsync(thr, dthr, 48, cudaMemcpyDeviceToHost, ctx.st));
    CUDA_TRY(cudaStreamSynchronize(ctx.st));
  }
  // thresholds are packed sums (~0: no pair reaches the bound -> empty range)
  if (need_thr[0]) pb.KL = thr[0] == ~0ull ? ~0ull : compact_word(thr[0], P);
  if (need_thr[1]) pb.KH = thr[1] == ~0ull ? ~0ull : compact_word(thr[1], P);
  pb.kmin = compact_word(thr[2] + thr[4], P);
  pb.kmax = compact_word(thr[3] + thr[5], P);
  return PGPU_OK;
}

// Small-product driver (kernel in small_path.cuh)
#include "small_driver.inc"

int copy_in(Ctx& ctx, const pgpu_poly* p, size_t csz, const pgpu_options& o, const uint64_t** exps,
            const void** coef) {
  if (o.inputs_on_device) {
    *exps = p->exps;
    *coef = p->coeffs;
    return PGPU_OK;
  }
  uint64_t* e;
  uint8_t* c;
  TRY(ctx.ar->alloc(&e, p->n));
  TRY(ctx.ar->alloc(&c, p->n * csz));
  CUDA_TRY(cudaMemcpyAsync(e, p->exps, p->n * 8, cudaMemcpyHostToDevice, ctx.st));
  CUDA_TRY(cudaMemcpyAsync(c, p->coeffs, p->n * csz, cudaMemcpyHostToDevice, ctx.st));
  *exps = e;
  *coef = c;
  return PGPU_OK;
}

constexpr size_t kSmallStage = 1 << 20;

// Small host operands: packed into the device's pinned staging buffer and sent
// in one copy.  The caller holds the device lock and every product ends with a
// stream synchronisation, so the buffer is free again when the next call starts.
int copy_in_small(Ctx& ctx, DeviceState& dev, const pgpu_poly* a, const pgpu_poly* b, size_t csz,
                  Problem* pb) {
  if (!dev.stage) CUDA_TRY(cudaMallocHost((void**)&dev.stage, kSmallStage));
  uint8_t* g_stage = dev.stage;
  const size_t ea = (size_t)a->n * 8, ca = (size_t)a->n * csz, eb = (size_t)b->n * 8, cb = (size_t)b->n * csz;
  // 16-byte aligned sections: exps a | coef a | exps b | coef b
  auto up = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t oa = 0, oca = up(ea), ob = oca + up(ca), ocb = ob + up(eb), tot = ocb + up(cb);
  memcpy(g_stage + oa, a->exps, ea);
  memcpy(g_stage + oca, a->coeffs, ca);
  memcpy(g_stage + ob, b->exps, eb);
  memcpy(g_stage + ocb, b->coeffs, cb);
  uint8_t* d;
  TRY(ctx.ar->alloc(&d, tot));
  CUDA_TRY(cudaMemcpyAsync(d, g_stage, tot, cudaMemcpyHostToDevice, ctx.st));
  pb->aexp = reinterpret_cast<const uint64_t*>(d + oa);
  pb->acoef = d + oca;
  pb->bexp = reinterpret_cast<const uint64_t*>(d + ob);
  pb->bcoef = d + ocb;
  return PGPU_OK;
}

int mul_impl(const pgpu_poly* a, const pgpu_poly* b, const pgpu_layout* lay,
             const pgpu_options* opt, pgpu_result* out) {
  if (!a || !b || !lay || !out) return fail(PGPU_EINVAL, "null argument");
  pgpu_options o;
  if (opt) o = *opt; else pgpu_default_options(&o);
  memset(out, 0, sizeof *out);
  out->coef_kind = o.coef_kind == PGPU_F64 ? PGPU_F64 : PGPU_I64;
  out->on_device = o.outputs_on_device;
  if (lay->nfields < 1 || lay->nfields > PGPU_MAX_FIELDS)
    return fail(PGPU_EINVAL, "layout needs 1..%d fields", PGPU_MAX_FIELDS);
  if (o.coef_kind < 0 || o.coef_kind > 2) return fail(PGPU_EINVAL, "unknown coefficient kind");
  if (a->n < 0 || b->n < 0 || a->n > 0xffffffffll || b->n > 0xffffffffll)
    return fail(PGPU_EINVAL, "operand sizes must be in [0, 2^32)");
  if (o.lo >= o.hi) return fail(PGPU_EINVAL, "empty exponent range");
  if (a->n == 0 || b->n == 0) return PGPU_OK;  // Polynomial.zero (parmul.py:102-103)

  g_trace.on = getenv("PGPU_TRACE") != nullptr;
  g_trace.n = 0;
  g_trace.at("entry");
  struct TraceDump {
    ~TraceDump() { g_trace.dump(); }
  } trace_dump;
  cudaStream_t lib_st;
  TRY(device_setup(o.device, &lib_st));
  Ctx ctx;
  ctx.st = o.stream ? (cudaStream_t)o.stream : lib_st;
  ctx.device = o.device;
  CUDA_TRY(cudaDeviceGetAttribute(&ctx.sms, cudaDevAttrMultiProcessorCount, o.device));
  DeviceState& dstate = g_dev[o.device & 63];
  ctx.rb = dstate.rb;
  std::lock_guard<std::mutex> ws_lock(dstate.mu);
  g_trace.at("setup");
  TRY(grow_workspace(dstate, ctx.st));
  g_trace.at("workspace");
  Arena ar(ctx.st, &dstate);
  ctx.ar = &ar;
  ctx.mem_budget = dstate.mem_free0 > dstate.ws_cap ? dstate.mem_free0 - dstate.ws_cap : 0;
  ctx.tm.start(ctx.st, o.timing != 0);

  Problem pb;
  memset(&pb, 0, sizeof pb);
  pb.ck = o.coef_kind;
  pb.na = (uint32_t)a->n;
  pb.nb = (uint32_t)b->n;
  size_t csz = o.coef_kind == PGPU_I128 ? 16 : 8;
  const size_t in_bytes = (size_t)(a->n + b->n) * (8 + csz);
  if (!o.inputs_on_device && in_bytes <= kSmallStage) {
    // small operands: one pinned staging buffer, one host-to-device copy
    TRY(copy_in_small(ctx, dstate, a, b, csz, &pb));
  } else {
    TRY(copy_in(ctx, a, csz, o, &pb.aexp, &pb.acoef));
    TRY(copy_in(ctx, b, csz, o, &pb.bexp, &pb.bcoef));
  }
  g_trace.at("copy_in");
  TRY(build_problem(ctx, lay, opt, pb, o));
  out->key_bits = pb.P.kbits;
  out->acc_limbs = pb.nl ? pb.nl : 1;

  // small products: one CTA, one launch, one host round trip
  if (pb.KL < pb.KH && (o.path == PGPU_PATH_AUTO || o.path == PGPU_PATH_SMALL) &&
      !getenv("PGPU_NO_SMALL")) {
    ctx.tm.mark(0, "prep");
    bool done = false;
    TRY(small_run(ctx, pb, o, out, &done));
    if (done) {
      ctx.tm.finish(out);
      CUDA_TRY(cudaGetLastError());
      out->kernel_launches = ctx.launches;
      return PGPU_OK;
    }
  }
  std::vector<Slice> slices;
  if (pb.KL < pb.KH) {
    // total pairs in range
    uint64_t total = (uint64_t)pb.na * pb.nb;
    if (o.range_pairs > 0) {
      total = (uint64_t)o.range_pairs;  // the caller's plan (a previous result's pair count)
    } else if (pb.KL > pb.kmin || pb.KH <= pb.kmax) {
      // pairs below both ends of the range in one count (one round trip)
      std::vector<uint64_t> bb{pb.KL}, cb;
      if (pb.KH != ~0ull) bb.push_back(pb.KH);
      if (pb.k32) TRY(count_at<uint32_t>(ctx, pb, bb, cb)); else TRY(count_at<uint64_t>(ctx, pb, bb, cb));
      const uint64_t below_hi = pb.KH != ~0ull ? cb[1] : (uint64_t)pb.na * pb.nb;
      total = below_hi - cb[0];
    }
    out->pairs = (int64_t)total;
    ctx.tm.mark(0, "prep");
    int path = o.path;
    // the reference's float order (merge.py:32-33): the bucket and sort paths
    // fold each term in increasing row; the dense path's warp copies do not
    const bool ordered = o.float_ordered && o.coef_kind == PGPU_F64;
    if (ordered && path == PGPU_PATH_DENSE)
      return fail(PGPU_EUNSUPPORTED, "float_ordered products do not take the dense path");
    int used = PGPU_PATH_SORT;
    if (path == PGPU_PATH_SMALL) path = PGPU_PATH_AUTO;  // product too large for one CTA
    if (path != PGPU_PATH_SORT && path != PGPU_PATH_BUCKET && !ordered) {
      int r = dense_try(ctx, pb, total, slices, path == PGPU_PATH_DENSE, &used);
      if (r != PGPU_OK) return r;
    }
    if (used == PGPU_PATH_SORT) {
      // sparse products: buckets per CTA; explicit PATH_SORT keeps the global
      // radix sort.  Products whose keys carry thousands of pairs (dense
      // products in the reference's float order) would overflow the buckets:
      // they go straight to the sort path.
      const uint64_t hiK = pb.KH == ~0ull ? pb.kmax + 1 : std::min(pb.KH, pb.kmax + 1);
      const uint64_t loK = std::max(pb.KL, pb.kmin);
      const bool dense_like = hiK > loK && hiK - loK <= 4 * total;  // the dense path's criterion
      // AUTO: buckets for products of up to 2^23 pairs (fewer launches); above
      // that the radix passes win (MP n=12, 3.8e7 pairs: sort 2.02 ms int /
      // 1.90 ms f64 against bucket 2.24 / 2.37 ms)
      const bool bucket = o.path != PGPU_PATH_SORT && !getenv("PGPU_NO_BUCKET") &&
                          !(ordered && o.path == PGPU_PATH_AUTO && dense_like) &&
                          (o.path == PGPU_PATH_BUCKET || total <= (1ull << 23));
      int nbucket = 0;
      int r = PGPU_OK;
      for (double scale = 1.0; scale >= 0.25; scale *= 0.5) {
        // out of memory (other users of the device): retry with smaller batches
        for (auto& sl : slices)
          for (void* q : {(void*)sl.exps, (void*)sl.coef})
            if (ar.owns(q)) {
              ar.release(q);
              cudaFreeAsync(q, ctx.st);
            }
        slices.clear();
        nbucket = 0;
        if (pb.k32) r = run_sort_path<uint32_t>(ctx, pb, total, slices, bucket, &nbucket, scale);
        else r = run_sort_path<uint64_t>(ctx, pb, total, slices, bucket, &nbucket, scale);
        if (r != PGPU_ENOMEM) break;
        cudaGetLastError();
        cudaStreamSynchronize(ctx.st);
      }
      TRY(r);
      if (nbucket > 0) used = PGPU_PATH_BUCKET;
    }
    out->path_used = used;
  }

  // assemble the result
  int nl = pb.nl ? pb.nl : 1;
  uint64_t n = 0;
  for (auto& s : slices) n += s.n;
  out->n = (int64_t)n;
  out->acc_limbs = nl;
  if (o.outputs_on_device) {
    uint64_t *e, *c;
    if (slices.size() == 1 && ar.owns(slices[0].exps) && ar.owns(slices[0].coef)) {
      e = slices[0].exps;
      c = slices[0].coef;
    } else {
      TRY(ar.alloc_out(&e, n));
      TRY(ar.alloc_out(&c, n * nl));
      uint64_t at = 0;
      for (auto& s : slices) {
        CUDA_TRY(cudaMemcpyAsync(e + at, s.exps, s.n * 8, cudaMemcpyDeviceToDevice, ctx.st));
        CUDA_TRY(cudaMemcpyAsync(c + at * nl, s.coef, s.n * 8 * nl, cudaMemcpyDeviceToDevice, ctx.st));
        at += s.n;
      }
    }
    ar.release(e);
    ar.release(c);
    out->exps = e;
    out->coeffs = c;
    out->_owner = (void*)(kDevTag | (uintptr_t)(o.device & 0xff));
  } else {
    out->exps = (uint64_t*)g_pinned.get(std::max<uint64_t>(n, 1) * 8);
    out->coeffs = g_pinned.get(std::max<uint64_t>(n, 1) * 8 * nl);
    out->_owner = (void*)kPinnedTag;
    if (!out->exps || !out->coeffs) return fail(PGPU_ENOMEM, "pinned host allocation failed");
    uint64_t at = 0;
    for (auto& s : slices) {
      CUDA_TRY(cudaMemcpyAsync(out->exps + at, s.exps, s.n * 8, cudaMemcpyDeviceToHost, ctx.st));
      CUDA_TRY(cudaMemcpyAsync((uint64_t*)out->coeffs + at * nl, s.coef, s.n * 8 * nl,
                               cudaMemcpyDeviceToHost, ctx.st));
      at += s.n;
    }
  }
  g_trace.at("output_launch");
  CUDA_TRY(cudaStreamSynchronize(ctx.st));
  g_trace.at("output_sync");
  ctx.tm.mark(5, "output");
  ctx.tm.finish(out);
  CUDA_TRY(cudaGetLastError());
  out->kernel_launches = ctx.launches;
  return PGPU_OK;
}

// PolyFile formatter driver (kernels in format.cuh, text.cuh)
#include "format_driver.inc"

}  // namespace

extern "C" {

void pgpu_default_options(pgpu_options* o) {
  memset(o, 0, sizeof *o);
  o->coef_kind = PGPU_F64;
  o->hi = ~0ull;
}

int pgpu_mul(const pgpu_poly* a, const pgpu_poly* b, const pgpu_layout* lay,
             const pgpu_options* opt, pgpu_result* out) {
  DeviceRestore dr;
  int r = mul_impl(a, b, lay, opt, out);
  if (r != PGPU_OK && out) {
    // release anything already handed to the result
    pgpu_free_result(out);
  }
  return r;
}

int pgpu_count_below(const pgpu_poly* a, const pgpu_poly* b, const pgpu_layout* lay,
                     const uint64_t* bounds, int64_t nbounds, const pgpu_options* opt,
                     uint64_t* cum) {
  if (!a || !b || !lay || !cum || (nbounds > 0 && !bounds)) return fail(PGPU_EINVAL, "null argument");
  pgpu_options o;
  if (opt) o = *opt; else pgpu_default_options(&o);
  if (nbounds <= 0) return PGPU_OK;
  if (a->n == 0 || b->n == 0) {
    for (int64_t k = 0; k < nbounds; ++k) cum[k] = 0;
    return PGPU_OK;
  }
  DeviceRestore dr;
  cudaStream_t lib_st;
  TRY(device_setup(o.device, &lib_st));
  Ctx ctx;
  ctx.st = o.stream ? (cudaStream_t)o.stream : lib_st;
  Arena ar(ctx.st);
  ctx.ar = &ar;
  Problem pb;
  memset(&pb, 0, sizeof pb);
  pb.na = (uint32_t)a->n;
  pb.nb = (uint32_t)b->n;
  size_t csz = o.coef_kind == PGPU_I128 ? 16 : 8;
  o.coef_kind = o.coef_kind;
  TRY(copy_in(ctx, a, csz, o, &pb.aexp, &pb.acoef));
  TRY(copy_in(ctx, b, csz, o, &pb.bexp, &pb.bcoef));
  // packed-space counting: the packed words themselves are the keys
  pb.ak = (void*)pb.aexp;
  pb.bk = (void*)pb.bexp;
  std::vector<uint64_t> bv(bounds, bounds + nbounds), cv;
  TRY(count_at<uint64_t>(ctx, pb, bv, cv));
  for (int64_t k = 0; k < nbounds; ++k) cum[k] = cv[k];
  return PGPU_OK;
}

void pgpu_free_result(pgpu_result* r) {
  if (!r) return;
  if (r->on_device) {
    // stream-ordered free on the owning device's stream: the memory goes back
    // to the (retained) pool for the next product instead of to the driver
    free_device_ptr(r->exps, r->_owner);
    free_device_ptr(r->coeffs, r->_owner);
  } else if (r->_owner == (void*)kPinnedTag) {
    if (r->exps) g_pinned.put(r->exps);
    if (r->coeffs) g_pinned.put(r->coeffs);
  } else {
    free(r->exps);
    free(r->coeffs);
  }
  r->exps = nullptr;
  r->coeffs = nullptr;
  r->n = 0;
}

int pgpu_format(const pgpu_poly* p, const pgpu_layout* lay, int64_t begin, int64_t end,
                const pgpu_options* opt, pgpu_text* out) {
  DeviceRestore dr;
  int r = format_impl(p, lay, begin, end, opt, out);
  if (r != PGPU_OK && out) pgpu_free_text(out);
  return r;
}

void pgpu_free_text(pgpu_text* t) {
  if (!t || !t->text) return;
  if (t->on_device) free_device_ptr(t->text, t->_owner);
  else if (t->_owner == (void*)kPinnedTag) g_pinned.put(t->text);
  else free(t->text);
  t->text = nullptr;
  t->bytes = 0;
}

int pgpu_ipc_alloc(int64_t bytes, int32_t device, void** dptr, void* handle) {
  if (!dptr || !handle || bytes < 0) return fail(PGPU_EINVAL, "null argument");
  DeviceRestore dr;
  CUDA_TRY(cudaSetDevice(device));
  *dptr = nullptr;
  // plain cudaMalloc: stream-ordered pool memory is not IPC-shareable by default
  CUDA_TRY(cudaMalloc(dptr, (size_t)std::max<int64_t>(bytes, 256)));
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, *dptr);
  if (e != cudaSuccess) {
    cudaFree(*dptr);
    *dptr = nullptr;
    return fail(PGPU_ECUDA, "cudaIpcGetMemHandle failed: %s", cudaGetErrorString(e));
  }
  static_assert(sizeof(h) <= PGPU_IPC_HANDLE_BYTES, "IPC handle size");
  memset(handle, 0, PGPU_IPC_HANDLE_BYTES);
  memcpy(handle, &h, sizeof h);
  return PGPU_OK;
}

int pgpu_ipc_open(const void* handle, int32_t device, void** dptr) {
  if (!dptr || !handle) return fail(PGPU_EINVAL, "null argument");
  DeviceRestore dr;
  CUDA_TRY(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  CUDA_TRY(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return PGPU_OK;
}

int pgpu_ipc_close(void* dptr) {
  CUDA_TRY(cudaIpcCloseMemHandle(dptr));
  return PGPU_OK;
}

int pgpu_ipc_free(void* dptr) {
  CUDA_TRY(cudaFree(dptr));
  return PGPU_OK;
}

int pgpu_copy(void* dst, const void* src, int64_t bytes, int32_t device, void* stream) {
  if (bytes <= 0) return PGPU_OK;
  if (!dst || !src) return fail(PGPU_EINVAL, "null argument");
  DeviceRestore dr;
  cudaStream_t lib_st;
  TRY(device_setup(device, &lib_st));
  CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice,
                           stream ? (cudaStream_t)stream : lib_st));
  return PGPU_OK;
}

int pgpu_stream_sync(int32_t device, void* stream) {
  DeviceRestore dr;
  cudaStream_t lib_st;
  TRY(device_setup(device, &lib_st));
  CUDA_TRY(cudaStreamSynchronize(stream ? (cudaStream_t)stream : lib_st));
  return PGPU_OK;
}

const char* pgpu_last_error(void) { return g_err.c_str(); }

int pgpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int pgpu_abi_version(void) { return PGPU_ABI_VERSION; }

}  // extern "C"
