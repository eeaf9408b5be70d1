// Device building blocks of the generic DFT engine (fft_generic.cu), shared
// with the single-CTA tail chains (real_fft.cu) so both run the same
// arithmetic: complex helpers, the shared-memory Stockham pass and one tile
// of the mixed-radix outer pass.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fgc_device.cuh"

namespace fgc {
namespace gdev {

template <class R> struct V2;
template <> struct V2<float> { using T = float2; };
template <> struct V2<double> { using T = double2; };

__device__ __forceinline__ float2 mk(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ double2 mk(double x, double y) { return make_double2(x, y); }

__device__ __forceinline__ float2 zmul(float2 a, float2 b) { return cmul(a, b); }
__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
template <class T2> __device__ __forceinline__ T2 zconj(T2 a) { return mk(a.x, -a.y); }
template <class T2> __device__ __forceinline__ T2 zadd(T2 a, T2 b) { return mk(a.x + b.x, a.y + b.y); }
template <class T2> __device__ __forceinline__ T2 zsub(T2 a, T2 b) { return mk(a.x - b.x, a.y - b.y); }


// W_S^j, j < 3S/4, from the global table of W_twP into shared memory (the
// same values; every stage reads its twiddles without an L2 round trip).
// Caller syncs.
constexpr uint32_t stage_twiddles(uint32_t S) { return S - (S >> 2); }
template <class T2>
__device__ __forceinline__ void load_stage_twiddles(T2* stw, uint32_t S, const T2* tw, uint32_t twP) {
  const uint32_t step = twP / S;
  for (uint32_t j = threadIdx.x; j < stage_twiddles(S); j += blockDim.x) stw[j] = tw[(uint64_t)j * step];
}

// Stockham autosort FFT over `nt` transforms of size S (a power of two)
// held in shared memory: one radix-2 stage when log2 S is odd, then radix-4
// stages (half the stages and barriers of radix-2; the quarter-turn of a
// radix-4 butterfly is exact).  stw = W_S^j (j < 3S/4) in shared memory.
template <class T2>
__device__ T2* smem_stockham(T2* x, T2* y, uint32_t S, uint32_t nt, const T2* stw, int dir) {
  const uint32_t lg = __ffs(S) - 1;
  uint32_t p = 1;
  if (lg & 1u) {                                      // radix-2 stage (p = 1: no twiddle)
    const uint32_t half = S >> 1;
    for (uint32_t b = threadIdx.x; b < nt * half; b += blockDim.x) {
      const uint32_t t = b >> (lg - 1), i = b & (half - 1);
      const T2 u0 = x[t * S + i], u1 = x[t * S + i + half];
      const uint32_t o = t * S + (i << 1);
      y[o] = zadd(u0, u1);
      y[o + 1] = zsub(u0, u1);
    }
    __syncthreads();
    T2* tmp = x; x = y; y = tmp;
    p = 2;
  }
  if (S < 4) return x;
  const uint32_t q4 = S >> 2, lq = lg - 2;
  for (; p < S; p <<= 2) {
    const uint32_t ts = S / (4 * p);
    for (uint32_t b = threadIdx.x; b < nt * q4; b += blockDim.x) {
      const uint32_t t = b >> lq, i = b & (q4 - 1);
      const uint32_t k = i & (p - 1);
      const T2* xs = x + t * S + i;
      const T2 x0 = xs[0];
      T2 w1 = stw[k * ts], w2 = stw[2 * k * ts], w3 = stw[3 * k * ts];
      if (dir > 0) { w1.y = -w1.y; w2.y = -w2.y; w3.y = -w3.y; }
      const T2 a1 = zmul(xs[q4], w1), a2 = zmul(xs[2 * q4], w2), a3 = zmul(xs[3 * q4], w3);
      const T2 t0 = zadd(x0, a2), t1 = zsub(x0, a2), t2 = zadd(a1, a3), d = zsub(a1, a3);
      const T2 t3 = dir < 0 ? mk(d.y, -d.x) : mk(-d.y, d.x);         // (a1 - a3) * (-+i)
      T2* yo = y + t * S + 4 * (i - k) + k;
      yo[0] = zadd(t0, t2);
      yo[p] = zadd(t1, t3);
      yo[2 * p] = zsub(t0, t2);
      yo[3 * p] = zsub(t1, t3);
    }
    __syncthreads();
    T2* tmp = x; x = y; y = tmp;
  }
  return x;
}

// Mixed-radix outer pass, Lc = A * B.  Index n = B n1 + n2, k = k1 + A k2.
//   forward (dir < 0): Y[k1 B + n2] = W^(k1 n2) sum_n1 x[B n1 + n2] W_A^(k1 n1)
//                      (then a B-point FFT down each row k1 gives X[k1 + A k2])
//   inverse (dir > 0): x[B n1 + n2] = sum_k1 W_A^(-k1 n1) (W^(-k1 n2) Y'[k1 B + n2])
//                      (after the B-point inverse FFT of each row k1)
// W = exp(-2 pi i / Lc) (exact table mtw), W_A = W^B.  A CTA takes `cols`
// columns n2 and `kg` output rows: the A x cols input tile (pre-twiddled for
// the inverse) and the A-entry W_A table sit in shared memory, so the A-term
// sums read no global memory.
// One tile (bx: column block, by: output-row block, item: batch entry) by
// the calling CTA, smem = (A + A * cols) entries; the caller syncs before
// reusing smem for another tile.
template <class T2>
__device__ __forceinline__ void mixed_tile(const T2* in, T2* out, const T2* mtw, uint32_t A, uint32_t B, uint32_t cols,
                                           uint32_t kg, int dir, uint32_t bx, uint32_t by, uint64_t item,
                                           unsigned char* smraw) {
  T2* wa = reinterpret_cast<T2*>(smraw);              // W_A^m (conjugated for the inverse), m < A
  T2* tile = wa + A;                                  // [A][cols]
  const uint32_t Lc = A * B;
  const uint32_t c0 = bx * cols, nc = min(cols, B - c0);
  const uint32_t o0 = by * kg, no = min(kg, A - o0);
  const T2* src = in + item * Lc;
  for (uint32_t m = threadIdx.x; m < A; m += blockDim.x) {
    T2 w = mtw[(uint64_t)m * B];
    if (dir > 0) w.y = -w.y;
    wa[m] = w;
  }
  for (uint32_t e = threadIdx.x; e < A * nc; e += blockDim.x) {
    const uint32_t i = e / nc, c = e - i * nc;
    T2 v = src[(uint64_t)i * B + c0 + c];
    if (dir > 0) {                                    // W^(-i n2); i n2 < 2^32 since Lc < 2^31
      T2 w = mtw[(uint32_t)(((uint64_t)i * (c0 + c)) % Lc)];
      w.y = -w.y;
      v = zmul(v, w);
    }
    tile[i * cols + c] = v;
  }
  __syncthreads();
  T2* dst = out + item * Lc;
  for (uint32_t e = threadIdx.x; e < no * nc; e += blockDim.x) {
    const uint32_t ol = e / nc, c = e - ol * nc, o = o0 + ol;
    // four independent partial sums (i mod 4) shorten the dependency chain
    T2 acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = mk(tile[0].x * 0, tile[0].y * 0);
    uint32_t m = 0;
    uint32_t i = 0;
    for (; i + 4 <= A; i += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc[u] = zadd(acc[u], zmul(tile[(i + u) * cols + c], wa[m]));
        m += o;
        if (m >= A) m -= A;
      }
    }
    for (; i < A; ++i) {
      acc[0] = zadd(acc[0], zmul(tile[i * cols + c], wa[m]));
      m += o;
      if (m >= A) m -= A;
    }
    T2 sum = zadd(zadd(acc[0], acc[1]), zadd(acc[2], acc[3]));
    if (dir < 0) sum = zmul(sum, mtw[(uint32_t)(((uint64_t)o * (c0 + c)) % Lc)]);   // W^(k1 n2)
    dst[(uint64_t)o * B + c0 + c] = sum;
  }
}


}  // namespace gdev
}  // namespace fgc
