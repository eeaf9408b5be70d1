// Register-resident FFT building blocks for the fused 65536-sample kernels.
//
// A CTA of 512 threads transforms M = 16384 complex points held 32 per
// thread in registers: three Stockham radix passes (32 x 32 x 16) with two
// shared-memory transposes between them (padded one float2 per 32 so every
// transpose is bank-conflict free).  Twiddles come from a two-level table of
// W_65536 = exp(-2 pi i / 65536) in shared memory (256 + 256 entries built in
// float64), so every twiddle costs one complex multiply.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fgc_device.cuh"

namespace fgc {
namespace ff {

constexpr int kThreads = 512;       // CTA size of the fused kernels
constexpr uint32_t kM = 16384;      // per-CTA transform length
constexpr uint32_t kN = 32768;      // complex length of a 65536-real chunk
constexpr uint32_t kL = 65536;      // chunk length
constexpr uint32_t kPadded = kM + kM / 32;

__device__ __forceinline__ uint32_t pad(uint32_t e) { return e + (e >> 5); }

// Twiddle tables in shared memory are stored with one spare entry per 8, so
// the strided lookups of the FFT passes (index j*k over the lanes k) spread
// over the banks: tpad(m) = m + m/8.
__host__ __device__ constexpr uint32_t tpad(uint32_t m) { return m + (m >> 3); }
constexpr uint32_t kTloPadded = 256 + 32;
constexpr uint32_t kT1024Padded = 1024 + 128;

// cos / sin (2 pi m / 32), m = 0..15
__device__ constexpr float kC32[16] = {1.0f, 0.98078528040323043f, 0.92387953251128674f, 0.83146961230254524f,
                                        0.70710678118654752f, 0.55557023301960222f, 0.38268343236508977f,
                                        0.19509032201612826f, 0.0f, -0.19509032201612826f, -0.38268343236508977f,
                                        -0.55557023301960222f, -0.70710678118654752f, -0.83146961230254524f,
                                        -0.92387953251128674f, -0.98078528040323043f};
__device__ constexpr float kS32[16] = {0.0f, 0.19509032201612826f, 0.38268343236508977f, 0.55557023301960222f,
                                        0.70710678118654752f, 0.83146961230254524f, 0.92387953251128674f,
                                        0.98078528040323043f, 1.0f, 0.98078528040323043f, 0.92387953251128674f,
                                        0.83146961230254524f, 0.70710678118654752f, 0.55557023301960222f,
                                        0.38268343236508977f, 0.19509032201612826f};

// cos / sin (2 pi m / 64), m = 0..31
__device__ constexpr float kC64[32] = {1.0f, 0.99518472667219693f, 0.98078528040323043f, 0.95694033573220882f, 0.92387953251128674f, 0.88192126434835505f, 0.83146961230254524f, 0.77301045336273699f, 0.70710678118654757f, 0.63439328416364549f, 0.55557023301960229f, 0.47139673682599781f, 0.38268343236508984f, 0.29028467725446233f, 0.19509032201612833f, 0.09801714032956077f, 6.123233995736766e-17f, -0.098017140329560645f, -0.19509032201612819f, -0.29028467725446216f, -0.38268343236508973f, -0.4713967368259977f, -0.55557023301960196f, -0.63439328416364538f, -0.70710678118654746f, -0.77301045336273699f, -0.83146961230254535f, -0.88192126434835494f, -0.92387953251128674f, -0.95694033573220882f, -0.98078528040323043f, -0.99518472667219682f};
__device__ constexpr float kS64[32] = {0.0f, 0.098017140329560604f, 0.19509032201612825f, 0.29028467725446233f, 0.38268343236508978f, 0.47139673682599764f, 0.55557023301960218f, 0.63439328416364549f, 0.70710678118654746f, 0.77301045336273699f, 0.83146961230254524f, 0.88192126434835494f, 0.92387953251128674f, 0.95694033573220894f, 0.98078528040323043f, 0.99518472667219682f, 1.0f, 0.99518472667219693f, 0.98078528040323043f, 0.95694033573220894f, 0.92387953251128674f, 0.88192126434835505f, 0.83146961230254546f, 0.7730104533627371f, 0.70710678118654757f, 0.63439328416364549f, 0.55557023301960218f, 0.47139673682599786f, 0.38268343236508989f, 0.29028467725446239f, 0.19509032201612861f, 0.098017140329560826f};

constexpr int bitrev(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}
constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

// d * W_32^m (forward: exp(-2 pi i m/32); INV: conjugate), m compile-time.
template <int M32, bool INV>
__device__ __forceinline__ float2 tw32(float2 d) {
  if constexpr (M32 == 0) {
    return d;
  } else if constexpr (M32 == 8) {
    return INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);
  } else {
    constexpr float c = kC32[M32];
    constexpr float s = INV ? kS32[M32] : -kS32[M32];
    return make_float2(__fmaf_rn(d.x, c, -d.y * s), __fmaf_rn(d.x, s, d.y * c));
  }
}

template <int S, int A, int R, bool INV>
__device__ __forceinline__ void dif_stage_inner(float2 (&v)[R]) {
  if constexpr (A < S) {
#pragma unroll
    for (int b = 0; b < R; b += 2 * S) {
      const float2 x = v[b + A], y = v[b + A + S];
      v[b + A] = make_float2(x.x + y.x, x.y + y.y);
      v[b + A + S] = tw32<A * (16 / S), INV>(make_float2(x.x - y.x, x.y - y.y));
    }
    dif_stage_inner<S, A + 1, R, INV>(v);
  }
}

template <int S, int R, bool INV>
__device__ __forceinline__ void dif_stages(float2 (&v)[R]) {
  if constexpr (S >= 1) {
    dif_stage_inner<S, 0, R, INV>(v);
    dif_stages<S / 2, R, INV>(v);
  }
}

// In-place radix-2 DIF DFT of R <= 32 points; result in bit-reversed order:
// v[bitrev(m)] = X[m].
template <int R, bool INV>
__device__ __forceinline__ void dft(float2 (&v)[R]) {
  static_assert(R == 16 || R == 32, "R");
  dif_stages<R / 2, R, INV>(v);
}

// d * W_64^J (forward), J < 32 compile-time.
template <int J>
__device__ __forceinline__ float2 w64mul(float2 d) {
  if constexpr (J == 0) {
    return d;
  } else if constexpr (J == 16) {
    return make_float2(d.y, -d.x);
  } else {
    constexpr float c = kC64[J];
    constexpr float s = -kS64[J];
    return make_float2(__fmaf_rn(d.x, c, -d.y * s), __fmaf_rn(d.x, s, d.y * c));
  }
}
// d * W_32^J (forward), J < 32 compile-time.
template <int J>
__device__ __forceinline__ float2 w32mul(float2 d) {
  if constexpr (J < 16) return w64mul<2 * J>(d);
  else return w64mul<2 * J - 32>(make_float2(-d.x, -d.y));
}

// W_65536^m from the two-level table (m taken mod 65536).
__device__ __forceinline__ float2 tw(const float2* thi, const float2* tlo, uint32_t m) {
  return cmul(thi[(m >> 8) & 255u], tlo[tpad(m & 255u)]);
}
__device__ __forceinline__ float2 twc(const float2* thi, const float2* tlo, uint32_t m, bool inv) {
  float2 w = tw(thi, tlo, m);
  if (inv) w.y = -w.y;
  return w;
}

// Passes 1 and 2 of the 16384-point transform.  On entry v[j] holds
// x[i + 512 j]; on exit the pass-2 output sits in `buf` (padded layout),
// ready for pass 3 (caller syncs).
template <bool INV>
__device__ __forceinline__ void fft_pass12(float2 (&v)[32], float2* buf, const float2* t1024) {
  const uint32_t i = threadIdx.x;
  dft<32, INV>(v);
  float2* w1 = buf + 33u * i;                           // pad(32 i + m) = 33 i + m
#pragma unroll
  for (int m = 0; m < 32; ++m) w1[m] = v[bitrev(m, 5)];
  __syncthreads();
  const float2* r2 = buf + i + (i >> 5);                // pad(i + 512 j) = i + i/32 + 528 j
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = r2[528 * j];
  const uint32_t k = i & 31u;
  // W_1024^{jk}: odd j from the table, even j as W^{(j-1)k} W^k -- half the
  // strided (bank-conflicting) table loads for one extra product
  const float2 wk = t1024[tpad(k)];
  float2 wprev = wk;
#pragma unroll
  for (int j = 1; j < 32; ++j) {
    float2 w;
    if (j & 1) {
      w = j == 1 ? wk : t1024[tpad(j * k)];
      wprev = w;
    } else {
      w = cmul(wprev, wk);
    }
    if (INV) w.y = -w.y;
    v[j] = cmul(v[j], w);
  }
  dft<32, INV>(v);
  float2* w2 = buf + (i >> 5) * 1056u + k;             // pad((i/32)*1024 + k + 32 m) = (i/32)*1056 + k + 33 m
  __syncthreads();                      // every pass-2 read is done before the writes
#pragma unroll
  for (int m = 0; m < 32; ++m) w2[33 * m] = v[bitrev(m, 5)];
}

// Pass 3 for one column k: reads x[k + 1024 j] (j < 16) from buf, applies
// W_16384^{jk}, and leaves out[m] = X[k + 1024 m] in natural order.
template <bool INV>
__device__ __forceinline__ void fft_pass3(uint32_t k, const float2* buf, float2 (&out)[16], const float2* thi,
                                          const float2* tlo) {
  float2 v[16];
  const float2* r3 = buf + k + (k >> 5);                // pad(k + 1024 j) = k + k/32 + 1056 j
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = r3[1056 * j];
  // W_16384^{jk}: odd j from the two-level table, even j as W^{(j-1)k} W^k
  const float2 wk = twc(thi, tlo, 4u * k, INV);
  float2 wprev = wk;
#pragma unroll
  for (int j = 1; j < 16; ++j) {
    float2 w;
    if (j & 1) {
      w = j == 1 ? wk : twc(thi, tlo, 4u * j * k, INV);
      wprev = w;
    } else {
      w = cmul(wprev, wk);
    }
    v[j] = cmul(v[j], w);
  }
  dft<16, INV>(v);
#pragma unroll
  for (int m = 0; m < 16; ++m) out[m] = v[bitrev(m, 4)];
}

}  // namespace ff
}  // namespace fgc
