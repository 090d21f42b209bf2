// format.cuh -- PolyFile text of a term range on the device (
// reference io.format_poly / write_poly, io.py:241-248, 306-308).
//
// Two passes over the terms, both HBM/latency-light integer work:
//   F1  FmtLen/FmtOff through device_scan: every term's line length (the
//       line is formatted into a counting writer), exclusive-scanned into
//       u64 byte offsets (offs[n] = total);
//   F2  k_fmt_write: one thread per term formats its line into the CTA's
//       shared-memory window, then the CTA stores the window's contiguous
//       bytes with aligned 4-byte stores (coalesced, instead of per-thread
//       scattered byte stores).
#pragma once
#include "scan.cuh"
#include "text.cuh"

namespace pgpu {

constexpr int kFmtThreads = 128;

struct FmtLen {
  const uint64_t* exps;
  const void* coef;
  text::LineSpec spec;
  __device__ uint64_t operator()(uint64_t i) const {
    text::CountW w;
    text::put_line(w, spec, exps[i], coef, i);
    return w.n;
  }
};

struct FmtOff {
  uint64_t* offs;
  uint64_t n;
  __device__ void operator()(uint64_t i, uint64_t ex, uint64_t v) const {
    offs[i] = ex;
    if (i + 1 == n) offs[n] = ex + v;
  }
};

__global__ void __launch_bounds__(kFmtThreads)
k_fmt_write(const uint64_t* __restrict__ exps, const void* __restrict__ coef, text::LineSpec spec,
            uint64_t n, const uint64_t* __restrict__ offs, char* __restrict__ out) {
  extern __shared__ __align__(16) char sbuf[];
  const uint64_t t0 = (uint64_t)blockIdx.x * kFmtThreads;
  if (t0 >= n) return;
  const uint64_t t1 = t0 + kFmtThreads < n ? t0 + kFmtThreads : n;
  const uint64_t base = offs[t0], endb = offs[t1];
  const uint64_t i = t0 + threadIdx.x;
  if (i < t1) {
    text::BufW w{sbuf + (offs[i] - base)};
    text::put_line(w, spec, exps[i], coef, i);
  }
  __syncthreads();
  const uint32_t len = (uint32_t)(endb - base);
  const uint32_t head = (uint32_t)((4 - (base & 3)) & 3) < len ? (uint32_t)((4 - (base & 3)) & 3) : len;
  if (threadIdx.x < head) out[base + threadIdx.x] = sbuf[threadIdx.x];
  const uint32_t words = (len - head) / 4;
  uint32_t* ow = reinterpret_cast<uint32_t*>(out + base + head);
  for (uint32_t k = threadIdx.x; k < words; k += kFmtThreads) {
    const char* s = sbuf + head + 4 * k;
    ow[k] = (uint32_t)(uint8_t)s[0] | ((uint32_t)(uint8_t)s[1] << 8) | ((uint32_t)(uint8_t)s[2] << 16) |
            ((uint32_t)(uint8_t)s[3] << 24);
  }
  const uint32_t tail0 = head + 4 * words;
  if (threadIdx.x < len - tail0) out[base + tail0 + threadIdx.x] = sbuf[tail0 + threadIdx.x];
}

}  // namespace pgpu
