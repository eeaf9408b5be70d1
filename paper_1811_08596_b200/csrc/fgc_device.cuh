// Device-side building blocks shared by every fgc kernel (sm_100a).
//
// Scalar semantics restate the reference exactly:
//   encode_code  <- quantizer.encode_array        (quantizer.py:217-236)
//                   + passthrough fold of -0.0     (codec.py:174-180)
//   decode_code  <- quantizer.decode_array        (quantizer.py:239-253)
//   cabs_key     <- np.abs(complex128), numpy's SIMD cabs (spectral.py:147)
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "fgc_types.h"

// Debug-only bounds checks (build with FGC_NVCC_FLAGS=-DFGC_BOUNDS).
#ifdef FGC_BOUNDS
#include <cstdio>
#define FGC_CHECK(cond)                                                                            \
  do {                                                                                             \
    if (!(cond)) {                                                                                 \
      printf("FGC_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x,   \
             threadIdx.x, #cond);                                                                  \
      __trap();                                                                                    \
    }                                                                                              \
  } while (0)
#else
#define FGC_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace fgc {

// ---------------------------------------------------------------- quantizer

__device__ __forceinline__ uint32_t encode_code(const QuantParams& q, float x) {
  if (q.n_bits == 32) return (x == 0.0f) ? 0u : __float_as_uint(x);
  const float a = fabsf(x);
  if (a < q.eps) return 0u;                       // codes[|x| < eps] = 0
  if (x > 0.0f) {
    uint32_t off = (__float_as_uint(fminf(a, q.pos_cap)) >> q.shift) - q.pbase + 1u;
    return min(off, q.npos);
  }
  uint32_t off = (__float_as_uint(fminf(a, q.neg_cap)) >> q.shift) - q.pbase + 1u;
  return q.npos + min(off, q.nneg);
}

__device__ __forceinline__ float decode_code(const QuantParams& q, uint32_t c) {
  if (q.n_bits == 32) return __uint_as_float(c);
  if (c == 0u) return 0.0f;
  if (c <= q.npos) return __uint_as_float((q.pbase + c - 1u) << q.shift);
  return -__uint_as_float((q.pbase + (c - q.npos) - 1u) << q.shift);
}

// ---------------------------------------------------------------- keys

// numpy's complex abs: larger * sqrt(fma(r, r, 1)), r = smaller/larger, 0/0 -> 0.
// Every operation is an explicit IEEE round-to-nearest intrinsic so nvcc
// cannot contract or approximate it.
__device__ __forceinline__ double cabs_key(double re, double im) {
  const double a = fabs(re), b = fabs(im);
  const double big = fmax(a, b), small = fmin(a, b);
  const double r = (big == 0.0) ? 0.0 : __ddiv_rn(small, big);
  return __dmul_rn(__dsqrt_rn(__fma_rn(r, r, 1.0)), big);
}

// Monotone fp32 proxy of the squared magnitude; within ~2 ulp of
// (cabs_key)^2 whenever it is a normal number far from over/underflow.
__device__ __forceinline__ float proxy_key(float re, float im) {
  return __fmaf_rn(re, re, __fmul_rn(im, im));
}

// ---------------------------------------------------------------- bits

// Wire bitmaps are MSB-first within each byte (packer.py:73-75); a warp
// ballot is LSB-first in slot order.  This involution converts between them.
__device__ __forceinline__ uint32_t ballot_to_wire(uint32_t w) {
  return __byte_perm(__brev(w), 0u, 0x0123);
}

// Spread the low 16 bits of x to the even bit positions.
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x &= 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

// Read `width` (<= 32) bits starting at bit `pos` of an LSB-first stream.
__device__ __forceinline__ uint32_t read_bits(const uint32_t* words, uint64_t pos, int width) {
  const uint64_t w = pos >> 5;
  const uint32_t o = (uint32_t)(pos & 31u);
  uint32_t lo = words[w];
  uint32_t v = lo >> o;
  if (o + (uint32_t)width > 32u) v |= words[w + 1] << (32u - o);
  return width == 32 ? v : (v & ((1u << width) - 1u));
}

// Release store of a completion tag (pairs with an ld.acquire.gpu spin).
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// A chunk's completion tag: system scope when peers on other GPUs read it.
__device__ __forceinline__ void release_tag(uint32_t* p, uint32_t v, uint32_t sys) {
  if (sys) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  } else {
    st_release_gpu(p, v);
  }
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- complex

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(__fmaf_rn(a.x, b.x, -a.y * b.y), __fmaf_rn(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {   // a * conj(b)
  return make_float2(__fmaf_rn(a.x, b.x, a.y * b.y), __fmaf_rn(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// ---------------------------------------------------------------- block scan

// Exclusive scan of one uint32 per thread across the block; returns the
// exclusive prefix and writes the block total.  `scratch` holds >= 33 words.
template <int THREADS>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* scratch, uint32_t& total) {
  static_assert(THREADS % 32 == 0 && THREADS <= 1024, "block size");
  constexpr int WARPS = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = (lane < WARPS) ? scratch[lane] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, d);
      if (lane >= d) s += y;
    }
    if (lane < WARPS) scratch[lane] = s;          // inclusive warp totals
    if (lane == 31) scratch[32] = s;
  }
  __syncthreads();
  const uint32_t base = warp ? scratch[warp - 1] : 0u;
  total = scratch[32];
  const uint32_t r = base + x - v;
  __syncthreads();                                // scratch reusable on return
  return r;
}

// Four independent exclusive scans at once (one set of barriers).
// `scratch` holds >= 4 * (THREADS / 32 + 1) words.
template <int THREADS>
__device__ __forceinline__ uint4 block_exclusive_scan4(uint4 v, uint32_t* scratch, uint4& total) {
  static_assert(THREADS % 32 == 0 && THREADS <= 512, "block size");
  constexpr int WARPS = THREADS / 32, S = WARPS + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x[k], d);
      if (lane >= d) x[k] += y;
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int k = 0; k < 4; ++k) scratch[k * S + warp] = x[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t s = (lane < WARPS) ? scratch[k * S + lane] : 0u;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, s, d);
        if (lane >= d) s += y;
      }
      if (lane < WARPS) scratch[k * S + lane] = s;   // inclusive warp totals; [WARPS-1] = block total
    }
  }
  __syncthreads();
  uint32_t out[4], tot[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    out[k] = (warp ? scratch[k * S + warp - 1] : 0u) + x[k] - (&v.x)[k];
    tot[k] = scratch[k * S + WARPS - 1];
  }
  total = make_uint4(tot[0], tot[1], tot[2], tot[3]);
  __syncthreads();
  return make_uint4(out[0], out[1], out[2], out[3]);
}

template <int THREADS>
__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t* scratch) {
  uint32_t total;
  block_exclusive_scan<THREADS>(v, scratch, total);
  return total;
}

}  // namespace fgc
